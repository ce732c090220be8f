// philox.cuh -- Philox-4x32-R on sm_100a.
//
// Same round function, output permutation and Weyl key schedule as the
// reference (proj/include/rgo/philox.hpp:46-96): R rounds, R-1 key bumps,
// p0 = M0*c0, p1 = M1*c2 (32x32->64), out = (hi1^c1^k0, lo1, hi0^c3^k1, lo0).
// Each 32x32->64 multiply is one IMAD.WIDE.U32; each 3-input xor one LOP3.
// Round keys depend only on the seed, so with a kernel-parameter key they
// live in uniform registers (UIADD3) and cost nothing per thread.
#pragma once
#include <cstdint>

namespace rgo_dev {

constexpr uint32_t kM0 = 0xD2511F53u;  // philox.hpp:46
constexpr uint32_t kM1 = 0xCD9E8D57u;  // philox.hpp:47
constexpr uint32_t kW0 = 0x9E3779B9u;  // philox.hpp:48
constexpr uint32_t kW1 = 0xBB67AE85u;  // philox.hpp:49

// philox_round, philox.hpp:54-62.
__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                             uint32_t& c3, uint32_t k0, uint32_t k1) {
    const uint64_t p0 = static_cast<uint64_t>(kM0) * c0;
    const uint64_t p1 = static_cast<uint64_t>(kM1) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = static_cast<uint32_t>(p1);
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = static_cast<uint32_t>(p0);
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
}

// philox_block with compile-time rounds, philox.hpp:84-96.
template <int R>
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        uint32_t k0, uint32_t k1) {
    static_assert(R >= 1 && R <= 16, "rounds must be in [1,16]");
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (r > 0) {
            k0 += kW0;
            k1 += kW1;
        }
        philox_round(c0, c1, c2, c3, k0, k1);
    }
    return make_uint4(c0, c1, c2, c3);
}

// Runtime-rounds variant (parity tests over R in [1,16]).
__device__ __forceinline__ uint4 philox_rt(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint32_t k0, uint32_t k1, int rounds) {
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) {
            k0 += kW0;
            k1 += kW1;
        }
        philox_round(c0, c1, c2, c3, k0, k1);
    }
    return make_uint4(c0, c1, c2, c3);
}

// Keep bits of one mask block counter: element_source (mask.hpp:72-85) maps
// the 64-bit counter base_offset + block to (c0, c1) = (lo, hi), c2 = c3 = 0;
// keeps() is word < threshold (mask.hpp:67), threshold < 2^32 here (the
// 2^32 "keep all" case is handled by the caller).  Returns 4 bits, LSB =
// lane 0 (mask.hpp:130, LSB-first packing).
template <int R>
__device__ __forceinline__ uint32_t keep4(uint64_t ctr, uint32_t k0, uint32_t k1, uint32_t thr) {
    const uint4 w = philox<R>(static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), 0u,
                              0u, k0, k1);
    return static_cast<uint32_t>(w.x < thr) | (static_cast<uint32_t>(w.y < thr) << 1) |
           (static_cast<uint32_t>(w.z < thr) << 2) | (static_cast<uint32_t>(w.w < thr) << 3);
}

// 32 keep bits = elements [32*q, 32*q+32) = 8 consecutive Philox blocks
// starting at counter ctr0 (bit j = element 32q+j, LSB-first).  General
// path: full 64-bit counter increment per block.
template <int R>
__device__ __forceinline__ uint32_t keep32(uint64_t ctr0, uint32_t k0, uint32_t k1, uint32_t thr) {
    uint32_t acc = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) acc |= keep4<R>(ctr0 + b, k0, k1, thr) << (4 * b);
    return acc;
}

// keep32 with runtime rounds (any R in [1,16]): the in-GEMM queue's drain for
// round counts without a compiled specialisation.
__device__ __forceinline__ uint32_t keep32_rt(uint64_t ctr0, uint32_t k0, uint32_t k1, uint32_t thr,
                                              int rounds) {
    uint32_t acc = 0;
#pragma unroll 1
    for (int b = 0; b < 8; ++b) {
        const uint64_t c = ctr0 + b;
        const uint4 w = philox_rt(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32), 0u, 0u, k0, k1, rounds);
        acc |= (static_cast<uint32_t>(w.x < thr) | (static_cast<uint32_t>(w.y < thr) << 1) |
                (static_cast<uint32_t>(w.z < thr) << 2) | (static_cast<uint32_t>(w.w < thr) << 3))
               << (4 * b);
    }
    return acc;
}

// acc = 2*acc + (w >= thr) in two ALU-pipe ops (IADD3 carry-out, IADD3.X):
// w - thr borrows exactly when w < thr, i.e. the carry-out is the DROP bit.
// `zero` is an opaque 0 (kernel parameter): the third addend keeps ptxas
// from lowering the carry-add to IMAD.X, which would land on the fma-heavy
// pipe that the IMAD.WIDE multiplies already saturate.  Callers feed
// elements high-to-low and invert once per 32-bit word.
__device__ __forceinline__ uint32_t push_drop_bit(uint32_t acc, uint32_t w, uint32_t thr,
                                                  uint32_t zero) {
    uint32_t r;
    asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 t, %3, %3;\n\tadd.u32 %0, t, %4;\n\t}"
        : "=r"(r)
        : "r"(w), "r"(thr), "r"(acc), "r"(zero));
    return r;
}

// Fast path when the low counter word cannot wrap inside the unit: c1 = hi is
// shared by all blocks, so round 1's c1^k0 and round 2's M0*(c1^k0) are
// computed once per thread instead of once per block (18 instead of 19
// IMAD.WIDE per block at R=10), and keep bits are packed with the carry
// chain above (2 ops/element).  Bit-identical to keep32().
template <int R>
__device__ __forceinline__ uint32_t keep32_nowrap(uint32_t lo, uint32_t hi, uint32_t k0,
                                                  uint32_t k1, uint32_t thr, uint32_t zero) {
    uint4 w[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) w[b] = philox<R>(lo + b, hi, 0u, 0u, k0, k1);
    uint32_t drop = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) {  // element 32q+4b+lane -> bit 4b+lane
        drop = push_drop_bit(drop, w[b].w, thr, zero);
        drop = push_drop_bit(drop, w[b].z, thr, zero);
        drop = push_drop_bit(drop, w[b].y, thr, zero);
        drop = push_drop_bit(drop, w[b].x, thr, zero);
    }
    return ~drop;
}

}  // namespace rgo_dev
