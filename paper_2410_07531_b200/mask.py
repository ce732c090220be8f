"""Dropout-mask API -- Python mirror of proj/include/rgo/mask.hpp.

Same names, argument meaning and exceptions (ValueError for the reference's
std::invalid_argument, RgoIOError for std::runtime_error).  Generation runs
on the GPU through the C ABI (K1, csrc/rng_mask.cu); only index arithmetic
(linear_index, element_source) and file I/O are host-side.
"""
from __future__ import annotations

import dataclasses
import math
import struct
from typing import Optional

import numpy as np

from . import _lib
from .philox import PhiloxCounter, PhiloxKey, philox_block

MAX_BITS = 1 << 36  # mask.hpp:108


@dataclasses.dataclass
class MaskLayout:  # mask.hpp:24-48
    batch: int = 1
    heads: int = 1
    seq: int = 1
    seed: int = 0
    base_offset: int = 0

    def elem_count(self) -> int:
        return self.batch * self.heads * self.seq * self.seq

    def linear_index(self, b: int, h: int, i: int, j: int) -> int:
        if b >= self.batch or h >= self.heads or i >= self.seq or j >= self.seq:
            raise ValueError("mask index out of range")
        return ((b * self.heads + h) * self.seq + i) * self.seq + j

    def key(self) -> PhiloxKey:
        return PhiloxKey(self.seed & 0xFFFFFFFF, (self.seed >> 32) & 0xFFFFFFFF)

    def validate(self) -> None:
        if self.elem_count() == 0:
            raise ValueError("mask layout has zero elements")


class KeepThreshold:  # mask.hpp:53-68
    def __init__(self, p: float):
        if not (0.0 <= p <= 1.0):
            raise ValueError("keep_prob must be in [0,1]")
        self.keep_prob = float(np.float32(p))  # stored as float, mask.hpp:59

    def threshold(self) -> int:
        # llround(double(float p) * 2^32), mask.hpp:62-65 (exact in binary64)
        x = self.keep_prob * 4294967296.0
        return int(math.floor(x + 0.5))

    def keeps(self, word: int) -> bool:
        return word < self.threshold()


def element_source(layout: MaskLayout, linear_index: int):
    """(counter, lane) for an element, mask.hpp:72-85 (64-bit wrap, c2=c3=0)."""
    if linear_index >= layout.elem_count():
        raise ValueError("element_source: linear index out of range")
    ctr = (layout.base_offset + (linear_index >> 2)) & 0xFFFFFFFFFFFFFFFF
    return PhiloxCounter(ctr & 0xFFFFFFFF, ctr >> 32, 0, 0), linear_index & 3


def keep_bit_direct(layout: MaskLayout, thr: KeepThreshold, rounds: int, linear_index: int) -> bool:
    """One keep bit straight from the PRNG (GPU philox_block), mask.hpp:88-92."""
    ctr, lane = element_source(layout, linear_index)
    return thr.keeps(philox_block(layout.key(), ctr, rounds).word(lane))


@dataclasses.dataclass
class DropoutMask:  # mask.hpp:94-105
    layout: MaskLayout = dataclasses.field(default_factory=MaskLayout)
    keep_prob: float = 1.0
    rounds: int = 7
    bits: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint8))

    def bit(self, b: int, h: int, i: int, j: int) -> bool:
        idx = self.layout.linear_index(b, h, i, j)
        return bool((int(self.bits[idx >> 3]) >> (idx & 7)) & 1)


def desc(layout: MaskLayout, thr: KeepThreshold, rounds: int) -> _lib.mask_desc:
    return _lib.mask_desc(
        layout.batch, layout.heads, layout.seq, rounds,
        layout.seed & 0xFFFFFFFFFFFFFFFF, layout.base_offset & 0xFFFFFFFFFFFFFFFF, thr.threshold(),
    )


def generate_mask(layout: MaskLayout, thr: KeepThreshold, rounds: int, workers: int = 0,
                  shards: int = 0) -> DropoutMask:
    """generate_mask, mask.hpp:142-179, on the GPU.  `workers` maps to the
    number of devices to shard over (0 = all); `shards` (>= devices) splits
    the mask into that many counter-offset shards, round-robin over the
    devices starting at the current one.  The bytes depend on neither
    (mask.hpp:139-141)."""
    layout.validate()
    if rounds < 1 or rounds > 16:
        raise ValueError("generate_mask: rounds must be in [1,16]")
    n = layout.elem_count()
    nbytes = (n + 7) // 8
    d = desc(layout, thr, rounds)
    if n > MAX_BITS:  # message produced by the C ABI (contains "bytes", "guard")
        _lib.check(_lib.lib().rgo_generate_mask_host(d, None, 0, 0))
    bits = np.empty(nbytes, dtype=np.uint8)
    _lib.check(_lib.lib().rgo_generate_mask_host_ex(d, bits.ctypes.data, nbytes, workers, shards))
    return DropoutMask(dataclasses.replace(layout), thr.keep_prob, rounds, bits)


def fnv1a64(data) -> int:
    """FNV-1a-64 of a host byte buffer (numpy / CPU tensor) via the C ABI."""
    arr = np.ascontiguousarray(data, dtype=np.uint8) if not hasattr(data, "numpy") else data.contiguous().numpy()
    return int(_lib.lib().rgo_fnv1a64(arr.ctypes.data, arr.size))


def generate_mask_device(layout: MaskLayout, thr: KeepThreshold, rounds: int, out=None,
                         stream=None, grid: int = 0, block: int = 0, dyn_smem: int = 0):
    """K1 into a device buffer (torch uint8 CUDA tensor), stream-ordered."""
    import torch

    layout.validate()
    nbytes = (layout.elem_count() + 7) // 8
    if out is None:
        out = torch.empty(((nbytes + 15) // 16) * 16, dtype=torch.uint8, device="cuda")
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    ls = _lib.launch(grid, block, dyn_smem, 0)
    _lib.check(_lib.lib().rgo_mask_generate_ex(desc(layout, thr, rounds), out.data_ptr(), out.numel(), ls, s))
    return out


def mask_bit(mask: DropoutMask, b: int, h: int, i: int, j: int) -> bool:
    """mask.hpp:183-186."""
    return mask.bit(b, h, i, j)


# --- RNGM file format (mask.hpp:188-297): 40-byte little-endian header + payload.
_HDR = struct.Struct("<4sHHIIIQQf")  # magic, version, rounds, B, nH, SQ, seed, base, keep_prob


def save_mask(mask: DropoutMask, path) -> None:
    hdr = _HDR.pack(b"RNGM", 1, mask.rounds, mask.layout.batch, mask.layout.heads, mask.layout.seq,
                    mask.layout.seed, mask.layout.base_offset, mask.keep_prob)
    try:
        with open(path, "wb") as f:
            f.write(hdr)
            f.write(np.ascontiguousarray(mask.bits, dtype=np.uint8).tobytes())
    except OSError as e:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"save_mask: cannot open {path}") from e


def load_mask(path) -> DropoutMask:
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: cannot open {path}") from e
    if len(raw) < _HDR.size:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: truncated header in {path}")
    magic, ver, rounds, b, h, s, seed, base, kp = _HDR.unpack_from(raw)
    if magic != b"RNGM":
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: bad magic in {path}")
    if ver != 1:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: unsupported version in {path}")
    layout = MaskLayout(b, h, s, seed, base)
    layout.validate()
    if rounds < 1 or rounds > 16:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: rounds out of range in {path}")
    n = layout.elem_count()
    nbytes = (n + 7) // 8
    payload = raw[_HDR.size:_HDR.size + nbytes]
    if len(payload) != nbytes:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: truncated payload in {path}")
    bits = np.frombuffer(payload, dtype=np.uint8).copy()
    if n % 8 and (int(bits[-1]) >> (n % 8)) != 0:
        raise _lib.RgoIOError(_lib.RGO_EIO, f"load_mask: nonzero padding bits in {path}")
    return DropoutMask(layout, float(np.float32(kp)), rounds, bits)
