"""Attention with dropout -- Python mirror of proj/include/rgo/ref_attention.hpp.

attention_forward / attention_dropout_fused / attention_dropout_decoupled keep
the reference's names, argument meaning and exceptions, and run the tcgen05
flash-attention kernel (csrc/attn_fwd_sm100.cu) through the C ABI
(rgo_attn_fwd).  Inputs are rounded to bf16 on the device (the tensor-core
dtype); outputs match the reference within the BF16 tolerance (5e-3), and the
fused and decoupled paths are bitwise equal to each other, as in the
reference (acceptance criterion 2).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List

import numpy as np

from . import _lib
from .mask import DropoutMask, KeepThreshold, MaskLayout, generate_mask

MASK_NONE, MASK_BITS, MASK_PHILOX = 0, 1, 2


@dataclasses.dataclass
class AttentionInput:  # ref_attention.hpp:21-41; q/k/v row-major (slice, pos, dim) float32
    slices: int = 1
    seq: int = 1
    head_dim: int = 1
    q: np.ndarray = None
    k: np.ndarray = None
    v: np.ndarray = None

    def elems(self) -> int:
        return self.slices * self.seq * self.head_dim

    def at(self, s: int, pos: int, d: int) -> int:
        return (s * self.seq + pos) * self.head_dim + d

    def scale(self) -> float:
        return float(np.float32(1.0) / np.sqrt(np.float32(self.head_dim)))

    def validate(self) -> None:
        if self.slices < 1 or self.seq < 1 or self.head_dim < 1:
            raise ValueError("attention dims must be >= 1")
        for x in (self.q, self.k, self.v):
            if x is None or x.size != self.elems():
                raise ValueError("attention input shape mismatch")


@dataclasses.dataclass
class AttentionOutput:  # ref_attention.hpp:43-48
    slices: int = 0
    seq: int = 0
    head_dim: int = 0
    o: np.ndarray = None

    def __eq__(self, other):
        return (self.slices, self.seq, self.head_dim) == (other.slices, other.seq, other.head_dim) and \
            np.array_equal(self.o.view(np.uint32), other.o.view(np.uint32))


def _padded_dim(d: int) -> int:
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise ValueError("head_dim > 128 is not supported by the tcgen05 kernel")


def _run_host(inp: AttentionInput, mask_source, keep_prob, bits, seed, base_offset, rounds):
    """head_dim > 128: the host entry point the C++ drop-in calls (rgo_attention_host),
    which runs the fp32 CUDA-core kernel K5g (csrc/attn_generic.cu) on the fp32 arrays."""
    import ctypes as C
    S, D, N = inp.seq, inp.head_dim, inp.slices
    q, k, v = (np.ascontiguousarray(x, np.float32) for x in (inp.q, inp.k, inp.v))
    o = np.empty(N * S * D, np.float32)
    b = np.ascontiguousarray(bits, np.uint8) if bits is not None else None
    ad = _lib.attn_host_desc(N, S, D, mask_source, float(keep_prob), seed, base_offset, rounds, 0)
    _lib.check(_lib.lib().rgo_attention_host(C.byref(ad), q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                             b.ctypes.data if b is not None else None,
                                             b.size if b is not None else 0, o.ctypes.data))
    return AttentionOutput(N, S, D, o)


def attn_fwd(q, k, v, o=None, *, mask_source=MASK_NONE, keep_prob=1.0, bits=None, seed=0, base_offset=0,
             rounds=10, scale=0.0, lse=None, stream=None):
    """Device-level K5/K6 on torch bf16 tensors shaped [B, H, S, D] (any
    strides with a contiguous D; D in {64, 128})."""
    import torch
    B, H, S, D = q.shape
    if o is None:
        o = torch.empty(B, H, S, D, dtype=torch.bfloat16, device=q.device)

    def t4(t):
        return _lib.tensor4(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))

    a = _lib.attn_desc(B, H, S, D, scale, mask_source, keep_prob, seed, base_offset, rounds, 0)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    _lib.check(_lib.lib().rgo_attn_fwd(a, t4(q), t4(k), t4(v), bits.data_ptr() if bits is not None else None,
                                       bits.numel() if bits is not None else 0, t4(o),
                                       lse.data_ptr() if lse is not None else None, s))
    return o


def attn_bwd(q, k, v, o, do, lse, *, mask_source=MASK_NONE, keep_prob=1.0, bits=None, seed=0, base_offset=0,
             rounds=10, scale=0.0, dq=None, dk=None, dv=None, work=None, stream=None, deterministic=False):
    """Device-level K7 (csrc/attn_bwd_sm100.cu): dQ, dK, dV (bf16 [B, H, S, D])
    of the K5/K6 forward with the same mask arguments; o and lse are that
    forward's output and natural-log LSE, do the incoming gradient.
    deterministic=True (head_dim 128): the split backward, dQ accumulated in
    TMEM with no cross-CTA reductions (bitwise reproducible, slower)."""
    import torch
    B, H, S, D = q.shape
    dev = q.device
    dq = torch.empty(B, H, S, D, dtype=torch.bfloat16, device=dev) if dq is None else dq
    dk = torch.empty(B, H, S, D, dtype=torch.bfloat16, device=dev) if dk is None else dk
    dv = torch.empty(B, H, S, D, dtype=torch.bfloat16, device=dev) if dv is None else dv

    def t4(t):
        return _lib.tensor4(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))

    a = _lib.attn_desc(B, H, S, D, scale, mask_source, keep_prob, seed, base_offset, rounds, 1 if deterministic else 0)
    need = _lib.C.c_uint64()
    _lib.check(_lib.lib().rgo_attn_bwd_workspace(a, _lib.C.byref(need)))
    if work is None or work.numel() * work.element_size() < need.value:
        work = torch.empty((need.value + 15) // 16 * 16, dtype=torch.uint8, device=dev)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    _lib.check(_lib.lib().rgo_attn_bwd(a, t4(q), t4(k), t4(v), t4(o), t4(do), lse.data_ptr(),
                                       bits.data_ptr() if bits is not None else None,
                                       bits.numel() if bits is not None else 0, t4(dq), t4(dk), t4(dv),
                                       work.data_ptr(), work.numel() * work.element_size(), s))
    return dq, dk, dv


class DropoutAttention:
    """torch.autograd.Function over K5/K6 (forward) and K7 (backward):
    ``DropoutAttention.apply(q, k, v, mask_source, keep_prob, bits, seed,
    base_offset, rounds)`` with bf16 [B, H, S, D] tensors.  The keep bits of
    the backward are the forward's (same mask buffer or Philox stream)."""

    _fn = None

    @classmethod
    def apply(cls, *args):
        if cls._fn is None:
            import torch

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, q, k, v, mask_source, keep_prob, bits, seed, base_offset, rounds):
                    B, H, S, D = q.shape
                    lse = torch.empty(B * H * S, dtype=torch.float32, device=q.device)
                    o = attn_fwd(q, k, v, mask_source=mask_source, keep_prob=keep_prob, bits=bits, seed=seed,
                                 base_offset=base_offset, rounds=rounds, lse=lse)
                    ctx.save_for_backward(q, k, v, o, lse, bits if bits is not None else torch.empty(0))
                    ctx.args = (mask_source, keep_prob, seed, base_offset, rounds, bits is not None)
                    return o

                @staticmethod
                def backward(ctx, do):
                    q, k, v, o, lse, bits = ctx.saved_tensors
                    mask_source, keep_prob, seed, base_offset, rounds, has_bits = ctx.args
                    dq, dk, dv = attn_bwd(q, k, v, o, do.contiguous(), lse, mask_source=mask_source,
                                          keep_prob=keep_prob, bits=bits if has_bits else None, seed=seed,
                                          base_offset=base_offset, rounds=rounds)
                    return dq, dk, dv, None, None, None, None, None, None

            cls._fn = _F
        return cls._fn.apply(*args)


def _run(inp: AttentionInput, mask_source, keep_prob=1.0, bits=None, seed=0, base_offset=0, rounds=7):
    import torch
    inp.validate()
    S, D, N = inp.seq, inp.head_dim, inp.slices
    if D > 128:
        return _run_host(inp, mask_source, keep_prob, bits, seed, base_offset, rounds)
    Dp = _padded_dim(D)
    dev = torch.device("cuda")

    def up(x):
        t = torch.zeros(1, N, S, Dp, dtype=torch.bfloat16, device=dev)
        t[..., :D] = torch.from_numpy(np.ascontiguousarray(x, np.float32)).view(1, N, S, D).to(dev)
        return t

    q, k, v = up(inp.q), up(inp.k), up(inp.v)
    dbits = None
    if bits is not None:
        nb = bits.size
        dbits = torch.zeros(((nb + 15) // 16) * 16, dtype=torch.uint8, device=dev)
        dbits[:nb] = torch.from_numpy(np.ascontiguousarray(bits, np.uint8)).to(dev)
    o = attn_fwd(q, k, v, mask_source=mask_source, keep_prob=keep_prob, bits=dbits, seed=seed,
                 base_offset=base_offset, rounds=rounds, scale=inp.scale())
    torch.cuda.synchronize()
    out = o[0, :, :, :D].float().cpu().numpy().reshape(-1)
    return AttentionOutput(N, S, D, np.ascontiguousarray(out))


def attention_forward(inp: AttentionInput) -> AttentionOutput:
    """Plain softmax(QK^T/sqrt(dH))V, ref_attention.hpp:108-110."""
    return _run(inp, MASK_NONE)


def attention_dropout_fused(inp: AttentionInput, seed: int, p: float, rounds: int,
                            base_offset: int = 0) -> AttentionOutput:
    """Keep bits regenerated inline (Philox in the attention kernel), ref_attention.hpp:114-126."""
    if not (0.0 < p <= 1.0):
        raise ValueError("attention_dropout_fused: p must be in (0,1]")
    if rounds < 1 or rounds > 16:
        raise ValueError("attention_dropout_fused: rounds must be in [1,16]")
    inp.validate()
    return _run(inp, MASK_PHILOX, p, seed=seed, base_offset=base_offset, rounds=rounds)


def attention_dropout_decoupled(inp: AttentionInput, mask: DropoutMask, p: float) -> AttentionOutput:
    """Keep bits read from a pre-generated mask, ref_attention.hpp:129-146."""
    if not (0.0 < p <= 1.0):
        raise ValueError("attention_dropout_decoupled: p must be in (0,1]")
    inp.validate()
    if mask.layout.batch * mask.layout.heads != inp.slices or mask.layout.seq != inp.seq:
        raise ValueError("attention_dropout_decoupled: mask layout mismatch")
    if float(np.float32(p)) != mask.keep_prob:
        raise ValueError("attention_dropout_decoupled: p mismatch with mask")
    return _run(inp, MASK_BITS, p, bits=mask.bits)


def random_attention_input(slices: int, seq: int, head_dim: int, seed: int) -> AttentionInput:
    """ref_attention.hpp:176-207, generated on the GPU (rgo_uniform_fill)."""
    import torch
    n = slices * seq * head_dim
    outs = []
    for stream_id in (1, 2, 3):
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().rgo_uniform_fill(seed & 0xFFFFFFFFFFFFFFFF, stream_id, n, None, t.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream))
        outs.append(t.cpu().numpy())
    return AttentionInput(slices, seq, head_dim, *outs)


@dataclasses.dataclass
class EquivCase:  # ref_attention.hpp:153-157
    slices: int
    seq: int
    head_dim: int
    seed: int
    p: float


@dataclasses.dataclass
class EquivResult:
    c: EquivCase
    bitwise_equal: bool = False


def default_equiv_grid() -> List[EquivCase]:
    """ref_attention.hpp:164-174."""
    cases, seed = [], 1000
    for (s, q, d) in ((1, 16, 8), (2, 64, 32), (4, 128, 64), (8, 256, 64)):
        for p in (0.5, 0.8, 0.9, 0.99):
            cases.append(EquivCase(s, q, d, seed, p))
            seed += 1
    return cases


def run_equiv_suite(cases: List[EquivCase], rounds: int = 7) -> List[EquivResult]:
    """ref_attention.hpp:209-227 on the GPU."""
    res = []
    for c in cases:
        inp = random_attention_input(c.slices, c.seq, c.head_dim, c.seed ^ 0xA77E)
        mask = generate_mask(MaskLayout(1, c.slices, c.seq, c.seed), KeepThreshold(c.p), rounds)
        fused = attention_dropout_fused(inp, c.seed, c.p, rounds)
        dec = attention_dropout_decoupled(inp, mask, c.p)
        res.append(EquivResult(c, fused == dec))
    return res
