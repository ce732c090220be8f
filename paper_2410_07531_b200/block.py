"""Transformer-block step (QKV/Proj/FFN GEMMs + attention with dropout) on
the B200 runtime (csrc/block.cu) through the C ABI (rgo_block_*).

Synthetic, random-init weights and activations of the named shape (no
checkpoints): values from the reference's Philox generator
(random_attention_input's counter layout, streams 4+), quantised per tensor
to E4M3.  Scales keep every intermediate O(1) so nothing saturates.
"""
from __future__ import annotations

import ctypes as C
import math

from . import _lib
from .gemm import WorkloadConfig
from .mask import KeepThreshold

MODES = {"serial_fused": 0, "streams": 1, "in_gemm": 2, "no_rng": 3}


def _uniform(n, stream_id, seed, device):
    import torch
    t = torch.empty(n, dtype=torch.float32, device=device)
    _lib.check(_lib.lib().rgo_uniform_fill(seed, stream_id, n, None, t.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
    return t


class Block:
    """Owns the device buffers of one block replica and the C-ABI handle."""

    def __init__(self, cfg: WorkloadConfig, mode: str = "streams", seed: int = 42, base_offset: int = 0,
                 rng_launch=(0, 0, 0), use_graph: bool = True, device="cuda", weights=None, chunks: int = 1,
                 chained: bool = False):
        """chunks > 1: SQ-chunk pipeline (pipeline_schedule, schedule.hpp:205-239): the
        query rows of every sequence split into `chunks` windows; a step is the rotation
        [attention(c) -> Proj/FFN1/FFN2/QKV of window c] over c, reading `qkv` (the
        previous step's QKV output) and writing `qkv_out`, with window c+1's mask hidden
        under stage c's GEMMs; the mask buffer is a 2-slot ring of window masks
        [slice][seq/chunks][seq] (2/chunks of the full mask).  chained=False (default):
        every step reads the same stationary input `attn_in` (unit-variance synthetic
        data); chained=True: each step consumes the previous step's attention output,
        which -- without the LayerNorm/residuals the reference also omits -- drifts to
        the e4m3 saturation limit over many steps."""
        import torch
        self.cfg, self.mode = cfg, mode
        B, S, H, D = cfg.batch, cfg.seq, cfg.heads, cfg.head_dim
        d, F = H * D, cfg.ffn()
        n1 = 2 * F if cfg.gated else F
        M = B * S
        self.M, self.d, self.F, self.n1 = M, d, F, n1
        f8, bf = torch.float8_e4m3fn, torch.bfloat16
        dev = torch.device(device)
        if weights is None:
            weights = make_weights(cfg, seed, dev)
        self.weights = weights
        self.x = _uniform(M * d, 8, seed, dev).view(M, d).to(f8)
        self.qkv = torch.empty(M, 3 * d, dtype=bf, device=dev)
        self.attn_in = _uniform(M * d, 9, seed, dev).view(M, d).mul_(math.sqrt(3.0)).to(bf)  # unit variance
        self.attn_o = self.attn_in.clone() if chained else torch.empty(M, d, dtype=bf, device=dev)
        self.attn_o8 = torch.empty(M, d, dtype=f8, device=dev)
        self.y1 = torch.empty(M, d, dtype=f8, device=dev)
        E, k = cfg.experts, cfg.top_k
        rows = M * k if E else M  # FFN rows: expert-sorted token copies for MoE
        self.h = torch.empty(rows, F, dtype=f8, device=dev)
        self.xd = torch.empty(rows, d, dtype=f8, device=dev) if E else None
        self.ye = torch.empty(rows, d, dtype=bf, device=dev) if E else None
        elems = B * H * S * S
        self.chunks = max(1, chunks)
        live = elems if self.chunks == 1 else 2 * (elems // self.chunks)
        self.mask = torch.zeros(live // 8, dtype=torch.uint8, device=dev)
        self.qkv_out = torch.empty(M, 3 * d, dtype=bf, device=dev) if self.chunks > 1 else None
        if self.chunks > 1:
            # the chunked step's input QKV: a deterministic synthetic stand-in for the
            # previous step's output (unit-variance Q/K/V), overwritten by callers at will
            self.qkv.copy_(_uniform(M * 3 * d, 10, seed, dev).view(M, 3 * d).mul_(math.sqrt(3.0)).to(bf))
        if mode == "no_rng" and self.chunks == 1:
            # NO_RNG never writes the mask; give its attention the real keep pattern
            # (an all-zero mask would feed the tensor cores zeros -- less power, higher
            # clock -- and make this measurement floor optimistic).  Chunked: the
            # runtime primes both ring slots with windows 0 and 1 on the first step.
            from .mask import MaskLayout, generate_mask_device
            lay = MaskLayout(B, H, S, seed, base_offset)
            generate_mask_device(lay, KeepThreshold(cfg.keep_prob), cfg.philox_rounds, out=self.mask)
            torch.cuda.synchronize()
        self.counter = torch.zeros(max(1, self.chunks), dtype=torch.int64, device=dev)
        self.lse = None
        # weights U(-1,1) (variance 1/3): alpha = sqrt(3/K) keeps activations at unit
        # variance; a chained step's input is an attention output (~0.1-0.3): s_attn 8
        desc = _lib.block_desc()
        desc.batch, desc.seq, desc.heads, desc.head_dim, desc.ffn = B, S, H, D, F
        desc.gated = 1 if cfg.gated else 0
        desc.keep_prob = cfg.keep_prob
        desc.rounds = cfg.philox_rounds
        desc.use_graph = 1 if use_graph else 0
        desc.seed, desc.base_offset = seed, base_offset
        desc.a_qkv, desc.a_proj = math.sqrt(3.0 / d), math.sqrt(3.0 / d)
        desc.a_ffn1, desc.a_ffn2 = math.sqrt(3.0 / d), math.sqrt(3.0 / F)
        desc.s_attn, desc.s_proj, desc.s_ffn1, desc.s_ffn2 = (8.0 if chained else 1.0), 1.0, 2.0, 1.0
        desc.rng_launch = _lib.launch(*rng_launch, 0)
        desc.experts, desc.top_k = (E, k) if E else (0, 0)
        desc.chunks = self.chunks
        self.desc = desc
        w = weights
        bufs = _lib.block_buffers(self.x.data_ptr(), w["wqkv"].data_ptr(), w["wo"].data_ptr(), w["w1"].data_ptr(),
                                  w["w2"].data_ptr(), self.qkv.data_ptr(), self.attn_o.data_ptr(),
                                  self.attn_o8.data_ptr(), self.y1.data_ptr(), self.h.data_ptr(),
                                  self.mask.data_ptr(), self.mask.numel(), self.counter.data_ptr(), None,
                                  self.xd.data_ptr() if E else None, self.ye.data_ptr() if E else None,
                                  None if chained else self.attn_in.data_ptr(),
                                  self.qkv_out.data_ptr() if self.qkv_out is not None else None)
        self._bufs = bufs
        handle = C.c_void_p()
        torch.cuda.synchronize()
        _lib.check(_lib.lib().rgo_block_create(desc, bufs, MODES[mode], C.byref(handle)))
        self.handle = handle

    def step(self, stream=None) -> int:
        import torch
        s = (stream or torch.cuda.current_stream()).cuda_stream
        n = C.c_int32()
        _lib.check(_lib.lib().rgo_block_step(self.handle, s, C.byref(n)))
        return n.value

    def last_timings(self):
        """(GEMM-window ms, attention ms) of the last completed step."""
        arr = (C.c_float * 2)()
        _lib.check(_lib.lib().rgo_block_last_timings(self.handle, arr))
        return float(arr[0]), float(arr[1])

    def last_timings3(self):
        """(GEMM window, RNG tail / join, attention kernel) ms of the last step."""
        arr = (C.c_float * 3)()
        _lib.check(_lib.lib().rgo_block_last_timings3(self.handle, arr))
        return float(arr[0]), float(arr[1]), float(arr[2])

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib().rgo_block_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_weights(cfg: WorkloadConfig, seed: int, device):
    import torch
    d, F = cfg.heads * cfg.head_dim, cfg.ffn()
    n1 = 2 * F if cfg.gated else F
    E = max(1, cfg.experts)  # MoE: experts stacked along the output rows
    f8 = torch.float8_e4m3fn
    return {
        "wqkv": _uniform(3 * d * d, 4, seed, device).view(3 * d, d).to(f8),
        "wo": _uniform(d * d, 5, seed, device).view(d, d).to(f8),
        "w1": _uniform(E * n1 * d, 6, seed, device).view(E * n1, d).to(f8),
        "w2": _uniform(E * d * F, 7, seed, device).view(E * d, F).to(f8),
    }
