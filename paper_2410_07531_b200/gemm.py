"""Block GEMMs (K2/K3/K4) -- the projections whose shapes the reference
defines in proj/include/rgo/workload.hpp:44-52 (QKV, Proj, FFN1, FFN2).

gemm_shapes/attention_work/rng_elements mirror the reference's arithmetic;
gemm() runs the hand-written tcgen05 kernel through the C ABI (rgo_gemm).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

from . import _lib

EPILOGUES = {"none": 0, "swiglu": 1, "gelu": 2}


@dataclasses.dataclass
class WorkloadConfig:  # workload.hpp:14-35 (+ ffn_dim / gated for Llama2-7B's 11008 SwiGLU FFN)
    batch: int = 1
    seq: int = 2048
    heads: int = 96
    head_dim: int = 128
    ffn_factor: int = 4
    precision_bytes: int = 1
    keep_prob: float = 0.9
    philox_rounds: int = 7
    ffn_dim: int = 0        # 0 = ffn_factor * hidden (reference formula)
    gated: bool = False     # SwiGLU: FFN1 has 2*ffn_dim outputs
    experts: int = 0        # MoE: number of expert FFNs (0 = dense FFN)
    top_k: int = 2          # MoE: experts per token

    def hidden(self) -> int:
        return self.heads * self.head_dim

    def ffn(self) -> int:
        return self.ffn_dim if self.ffn_dim else self.ffn_factor * self.hidden()

    def validate(self) -> None:
        if min(self.batch, self.seq, self.heads, self.head_dim, self.ffn_factor, self.precision_bytes) < 1:
            raise ValueError("workload dimensions must be >= 1")
        if not (0.0 <= self.keep_prob <= 1.0):
            raise ValueError("keep_prob must be in [0,1]")
        if not (1 <= self.philox_rounds <= 16):
            raise ValueError("philox_rounds must be in [1,16]")


@dataclasses.dataclass
class GemmShape:  # workload.hpp:37-42
    name: str
    m: int = 1
    n: int = 1
    k: int = 1

    def flops(self) -> int:
        return 2 * self.m * self.n * self.k


def gemm_shapes(cfg: WorkloadConfig) -> List[GemmShape]:
    """workload.hpp:44-52; with gated=True FFN1 is the fused gate+up GEMM."""
    cfg.validate()
    rows, h, f = cfg.batch * cfg.seq, cfg.hidden(), cfg.ffn()
    out = [GemmShape("QKV", rows, 3 * h, h), GemmShape("Proj", rows, h, h)]
    if cfg.experts:  # MoE: each expert sees rows*top_k/experts tokens (balanced routing)
        me = rows * cfg.top_k // cfg.experts
        for e in range(cfg.experts):
            out += [GemmShape(f"FFN1.e{e}", me, (2 if cfg.gated else 1) * f, h), GemmShape(f"FFN2.e{e}", me, h, f)]
        return out
    return out + [GemmShape("FFN1", rows, (2 if cfg.gated else 1) * f, h), GemmShape("FFN2", rows, h, f)]


def attention_work(cfg: WorkloadConfig):
    """workload.hpp:54-64: (mma_flops, softmax_elems)."""
    cfg.validate()
    elems = cfg.batch * cfg.heads * cfg.seq * cfg.seq
    return 4 * elems * cfg.head_dim, elems


def rng_elements(cfg: WorkloadConfig) -> int:
    """workload.hpp:66-70."""
    cfg.validate()
    return cfg.batch * cfg.heads * cfg.seq * cfg.seq


def workload_preset(name: str) -> WorkloadConfig:
    """workload.hpp:74-89, plus the BASELINE.json Llama2-7B block."""
    if name == "gpt3":
        return WorkloadConfig(seq=2048, heads=96)
    if name == "llama2":
        return WorkloadConfig(seq=4096, heads=64)
    if name == "moe":  # BASELINE configs[3]; shape chosen per SURVEY 8(d): Mixtral-8x7B-like
        return WorkloadConfig(batch=4, seq=4096, heads=32, head_dim=128, ffn_dim=14336, gated=True,
                              keep_prob=0.9, philox_rounds=10, experts=8, top_k=2)
    if name == "llama2_7b":
        return WorkloadConfig(batch=4, seq=4096, heads=32, head_dim=128, ffn_dim=11008, gated=True,
                              keep_prob=0.9, philox_rounds=10)
    raise ValueError(f"unknown workload preset '{name}' (known: gpt3, llama2, llama2_7b, moe)")


def _dt(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return 0
    if t.dtype in (torch.float8_e4m3fn, torch.uint8):
        return 1
    raise ValueError(f"unsupported dtype {t.dtype}")


def gemm_desc(a, b, c, alpha=1.0, out_scale=1.0, epilogue="none", grid=0) -> _lib.gemm_desc:
    return _lib.gemm_desc(a.shape[0], b.shape[0], a.shape[1], _dt(a), _dt(c), EPILOGUES[epilogue],
                          a.stride(0), b.stride(0), c.stride(0), alpha, out_scale, grid, 0)


def gemm(a, b, c=None, *, alpha: float = 1.0, out_scale: float = 1.0, epilogue: str = "none",
         out_dtype=None, grid: int = 0, stream=None):
    """c = epilogue(alpha * a @ b.T) * out_scale on the tensor cores.
    a: [M, K], b: [N, K] (bf16 or float8_e4m3fn, K-major); c: [M, N'] bf16/e4m3."""
    import torch
    if c is None:
        n_out = b.shape[0] // 2 if epilogue == "swiglu" else b.shape[0]
        c = torch.empty(a.shape[0], n_out, dtype=out_dtype or torch.bfloat16, device=a.device)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    d = gemm_desc(a, b, c, alpha, out_scale, epilogue, grid)
    _lib.check(_lib.lib().rgo_gemm(d, a.data_ptr(), b.data_ptr(), c.data_ptr(), s))
    return c


def gemm_with_rng(a, b, c, mask_desc: _lib.mask_desc, bits, counter, *, alpha: float = 1.0,
                  out_scale: float = 1.0, epilogue: str = "none", grid: int = 0, rng_warps: int = 0,
                  stream=None):
    """K4: gemm() with co-resident RNG warps (rng_warps per CTA: 4/6/8/12/16, 0 = 8)
    draining the mask queue."""
    import torch
    s = (stream or torch.cuda.current_stream()).cuda_stream
    d = gemm_desc(a, b, c, alpha, out_scale, epilogue, grid)
    d.rng_warps = rng_warps
    _lib.check(_lib.lib().rgo_gemm_with_rng(d, a.data_ptr(), b.data_ptr(), c.data_ptr(), mask_desc,
                                            bits.data_ptr(), bits.numel(), counter.data_ptr(), s))
    return c


def mask_queue_drain(mask_desc: _lib.mask_desc, bits, counter, grid=0, block=0, dyn_smem=0, stream=None):
    import torch
    s = (stream or torch.cuda.current_stream()).cuda_stream
    _lib.check(_lib.lib().rgo_mask_queue_drain(mask_desc, bits.data_ptr(), bits.numel(), counter.data_ptr(),
                                               _lib.launch(grid, block, dyn_smem, 0), s))
