"""Philox-4x32-R -- Python mirror of proj/include/rgo/philox.hpp.

philox_block / philox_round run on the GPU through the C ABI
(rgo_philox_blocks); bump_key and advance are the reference's plain counter
arithmetic (philox.hpp:65-80) and stay host-side integer helpers.
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np

from . import _lib

MULT0, MULT1 = 0xD2511F53, 0xCD9E8D57  # philox.hpp:46-47
WEYL0, WEYL1 = 0x9E3779B9, 0xBB67AE85  # philox.hpp:48-49
_M32 = 0xFFFFFFFF


class PhiloxKey(NamedTuple):  # philox.hpp:14-18
    k0: int = 0
    k1: int = 0


class PhiloxCounter(NamedTuple):  # philox.hpp:20-26
    c0: int = 0
    c1: int = 0
    c2: int = 0
    c3: int = 0


class PhiloxBlock(NamedTuple):  # philox.hpp:28-43
    w0: int = 0
    w1: int = 0
    w2: int = 0
    w3: int = 0

    def word(self, lane: int) -> int:
        return (self.w0, self.w1, self.w2)[lane] if lane < 3 else self.w3


def bump_key(key: PhiloxKey) -> PhiloxKey:
    """Weyl key step, philox.hpp:65-67."""
    return PhiloxKey((key.k0 + WEYL0) & _M32, (key.k1 + WEYL1) & _M32)


def advance(c: PhiloxCounter, n: int) -> PhiloxCounter:
    """128-bit counter += n with carry c0->c1->c2->c3, philox.hpp:70-80."""
    lo, hi = n & _M32, (n >> 32) & _M32
    c0 = (c.c0 + lo) & _M32
    if c0 < lo:
        hi = (hi + 1) & _M32  # uint32 ++hi wraps, exactly as the reference
    c1 = (c.c1 + hi) & _M32
    c2, c3 = c.c2, c.c3
    if c1 < hi:
        c2 = (c2 + 1) & _M32
        if c2 == 0:
            c3 = (c3 + 1) & _M32
    return PhiloxCounter(c0, c1, c2, c3)


def philox_blocks(keys: np.ndarray, ctrs: np.ndarray, rounds) -> np.ndarray:
    """Batched philox_block on the GPU: keys (n,2) u32, ctrs (n,4) u32,
    rounds scalar or (n,) -> (n,4) u32.  Rounds outside [1,16] raise
    ValueError like philox.hpp:86-87."""
    import torch

    keys = np.ascontiguousarray(keys, dtype=np.uint32).reshape(-1, 2)
    ctrs = np.ascontiguousarray(ctrs, dtype=np.uint32).reshape(-1, 4)
    n = keys.shape[0]
    r = np.broadcast_to(np.asarray(rounds, dtype=np.int32), (n,)).copy()
    if n and (r.min() < 1 or r.max() > 16):
        raise ValueError("philox_block: rounds must be in [1,16]")
    dev = torch.device("cuda")
    dk = torch.from_numpy(keys.view(np.int32)).to(dev)
    dc = torch.from_numpy(ctrs.view(np.int32)).to(dev)
    dr = torch.from_numpy(r).to(dev)
    out = torch.empty((n, 4), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(
        _lib.lib().rgo_philox_blocks(dk.data_ptr(), dc.data_ptr(), dr.data_ptr(), out.data_ptr(), n, stream)
    )
    return out.cpu().numpy().view(np.uint32)


def philox_block(key: PhiloxKey, counter: PhiloxCounter, rounds: int) -> PhiloxBlock:
    """philox_block(key, counter, rounds), philox.hpp:84-96 (GPU)."""
    if rounds < 1 or rounds > 16:
        raise ValueError("philox_block: rounds must be in [1,16]")
    out = philox_blocks(np.array([key], dtype=np.uint32), np.array([counter], dtype=np.uint32), rounds)
    return PhiloxBlock(*(int(x) for x in out[0]))


def philox_round(s: PhiloxCounter, key: PhiloxKey) -> PhiloxCounter:
    """One S-P round, philox.hpp:54-62 (= philox_block with rounds=1)."""
    return PhiloxCounter(*philox_block(key, s, 1))
