"""ctypes binding of the C-ABI boundary (include/rgo/capi.h).

The shared library is built in-tree (paper_2410_07531_b200/librgo_b200.so,
see csrc/Makefile).  Loading fails loudly when it is missing: there is no
CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# RGO_LIB_PATH: A/B measurements of an alternative build (scripts/diag)
LIB_PATH = os.environ.get("RGO_LIB_PATH") or os.path.join(_HERE, "librgo_b200.so")

RGO_OK, RGO_EINVAL, RGO_ECUDA, RGO_ENOMEM, RGO_EIO, RGO_ENODEV = range(6)


class RgoError(RuntimeError):
    """Non-validation failure (CUDA, device, allocation)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class RgoIOError(RgoError):
    """Mirror of the reference's std::runtime_error for mask file I/O."""


class mask_desc(C.Structure):
    _fields_ = [
        ("batch", C.c_uint32),
        ("heads", C.c_uint32),
        ("seq", C.c_uint32),
        ("rounds", C.c_uint32),
        ("seed", C.c_uint64),
        ("base_offset", C.c_uint64),
        ("threshold", C.c_uint64),
    ]


class launch(C.Structure):
    _fields_ = [
        ("grid", C.c_uint32),
        ("block", C.c_uint32),
        ("dyn_smem", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class gemm_desc(C.Structure):
    _fields_ = [
        ("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
        ("in_dtype", C.c_int32), ("out_dtype", C.c_int32), ("epilogue", C.c_int32),
        ("lda", C.c_int64), ("ldb", C.c_int64), ("ldc", C.c_int64),
        ("alpha", C.c_float), ("out_scale", C.c_float),
        ("grid", C.c_int32), ("rng_warps", C.c_int32),
    ]


class tensor4(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("stride_b", C.c_int64), ("stride_h", C.c_int64), ("stride_s", C.c_int64)]


class attn_desc(C.Structure):
    _fields_ = [
        ("batch", C.c_uint32), ("heads", C.c_uint32), ("seq", C.c_uint32), ("head_dim", C.c_uint32),
        ("scale", C.c_float), ("mask_source", C.c_int32), ("keep_prob", C.c_double),
        ("seed", C.c_uint64), ("base_offset", C.c_uint64), ("rounds", C.c_uint32), ("flags", C.c_uint32),
    ]


class attn_host_desc(C.Structure):
    _fields_ = [
        ("slices", C.c_uint32), ("seq", C.c_uint32), ("head_dim", C.c_uint32), ("mask_source", C.c_int32),
        ("keep_prob", C.c_double), ("seed", C.c_uint64), ("base_offset", C.c_uint64), ("rounds", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class block_desc(C.Structure):
    _fields_ = [
        ("batch", C.c_uint32), ("seq", C.c_uint32), ("heads", C.c_uint32), ("head_dim", C.c_uint32),
        ("ffn", C.c_uint32), ("gated", C.c_int32), ("keep_prob", C.c_double), ("rounds", C.c_uint32),
        ("use_graph", C.c_uint32), ("seed", C.c_uint64), ("base_offset", C.c_uint64),
        ("a_qkv", C.c_float), ("a_proj", C.c_float), ("a_ffn1", C.c_float), ("a_ffn2", C.c_float),
        ("s_attn", C.c_float), ("s_proj", C.c_float), ("s_ffn1", C.c_float), ("s_ffn2", C.c_float),
        ("rng_launch", launch), ("experts", C.c_uint32), ("top_k", C.c_uint32),
        ("chunks", C.c_uint32), ("reserved2", C.c_uint32),
    ]


class block_tp(C.Structure):
    _fields_ = [("size", C.c_uint32), ("rank", C.c_uint32), ("peer_part", C.c_void_p * 8),
                ("peer_y1", C.c_void_p * 8), ("peer_x", C.c_void_p * 8)]


BARRIER_FN = C.CFUNCTYPE(None, C.c_void_p)


class block_buffers(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("x", "wqkv", "wo", "w1", "w2", "qkv", "attn_o", "attn_o8", "y1", "h",
                                          "mask")] + [("mask_bytes", C.c_uint64), ("counter", C.c_void_p),
                                                      ("lse", C.c_void_p), ("xd", C.c_void_p), ("ye", C.c_void_p),
                                                      ("attn_in", C.c_void_p), ("qkv_out", C.c_void_p)]


# name -> (restype, argtypes).  Every symbol include/rgo/capi.h declares.
SIGNATURES = {
    "rgo_last_error": (C.c_char_p, []),
    "rgo_version": (C.c_int, []),
    "rgo_device_count": (C.c_int, []),
    "rgo_philox_blocks": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p],
    ),
    "rgo_keep_threshold": (C.c_int, [C.c_double, C.POINTER(C.c_uint64), C.POINTER(C.c_float)]),
    "rgo_mask_bytes": (C.c_int, [C.POINTER(mask_desc), C.POINTER(C.c_uint64)]),
    "rgo_mask_generate": (C.c_int, [C.POINTER(mask_desc), C.c_void_p, C.c_uint64, C.c_void_p]),
    "rgo_mask_generate_ex": (
        C.c_int,
        [C.POINTER(mask_desc), C.c_void_p, C.c_uint64, C.POINTER(launch), C.c_void_p],
    ),
    "rgo_generate_mask_host": (
        C.c_int,
        [C.POINTER(mask_desc), C.c_void_p, C.c_uint64, C.c_uint32],
    ),
    "rgo_generate_mask_host_ex": (
        C.c_int,
        [C.POINTER(mask_desc), C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32],
    ),
    "rgo_fnv1a64": (C.c_uint64, [C.c_void_p, C.c_uint64]),
    "rgo_mask_queue_drain": (
        C.c_int,
        [C.POINTER(mask_desc), C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(launch), C.c_void_p],
    ),
    "rgo_gemm": (C.c_int, [C.POINTER(gemm_desc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rgo_gemm_with_rng": (
        C.c_int,
        [C.POINTER(gemm_desc), C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(mask_desc), C.c_void_p,
         C.c_uint64, C.c_void_p, C.c_void_p],
    ),
    "rgo_attn_fwd": (
        C.c_int,
        [C.POINTER(attn_desc), C.POINTER(tensor4), C.POINTER(tensor4), C.POINTER(tensor4), C.c_void_p,
         C.c_uint64, C.POINTER(tensor4), C.c_void_p, C.c_void_p],
    ),
    "rgo_attn_bwd_workspace": (C.c_int, [C.POINTER(attn_desc), C.POINTER(C.c_uint64)]),
    "rgo_attn_bwd": (
        C.c_int,
        [C.POINTER(attn_desc)] + [C.POINTER(tensor4)] * 5 + [C.c_void_p, C.c_void_p, C.c_uint64]
        + [C.POINTER(tensor4)] * 3 + [C.c_void_p, C.c_uint64, C.c_void_p],
    ),
    "rgo_block_create": (C.c_int, [C.POINTER(block_desc), C.POINTER(block_buffers), C.c_int32, C.c_void_p]),
    "rgo_block_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "rgo_block_last_timings": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rgo_block_last_timings3": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rgo_block_destroy": (C.c_int, [C.c_void_p]),
    "rgo_block_create_tp": (C.c_int, [C.POINTER(block_desc), C.POINTER(block_buffers), C.c_void_p, C.c_int32,
                                      C.c_void_p]),
    "rgo_block_step_tp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rgo_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "rgo_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "rgo_ipc_close": (C.c_int, [C.c_void_p]),
    "rgo_philox_blocks_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    "rgo_random_attention_input_host": (
        C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rgo_attention_host": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "rgo_mask_save": (C.c_int, [C.c_char_p, C.POINTER(mask_desc), C.c_float, C.c_void_p, C.c_uint64]),
    "rgo_mask_load": (
        C.c_int, [C.c_char_p, C.POINTER(mask_desc), C.POINTER(C.c_float), C.c_void_p, C.c_uint64,
                  C.POINTER(C.c_uint64)]),
    "rgo_uniform_fill": (
        C.c_int,
        [C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
}

_lib = None


def lib() -> C.CDLL:
    """Load (once) the product library; raise if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2410_07531_b200/csrc` "
                "(or __graft_entry__.build()); the rgo B200 path has no CPU fallback"
            )
        dll = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        _lib = dll
    return _lib


def check(code: int) -> None:
    """Map an rgo_status to the reference's exception types."""
    if code == RGO_OK:
        return
    msg = lib().rgo_last_error().decode(errors="replace")
    if code == RGO_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if code == RGO_EIO:
        raise RgoIOError(code, msg)  # std::runtime_error
    raise RgoError(code, msg)
