// rng_queue.cuh -- dropout-mask work queue (overlap mechanism B).
// Warps claim 64-vector chunks (two 128-element vectors per lane) from a
// global counter; the same device routine runs inside the GEMM CTAs
// (co-resident RNG warps, until the GEMM's epilogue warps finish) and in the
// tail kernel that drains whatever the GEMMs left.  Bits are identical to K1:
// vector v = elements [128v, 128v+128), counter base + 32v (of the full
// layout's vector window_vec(win, v) when the queue covers a row window).
#pragma once
#include <cstdint>

#include "gemm.h"
#include "philox.cuh"

namespace rgo {

// k0/k1/thr arrive as per-thread (vector-register) copies: see rng_drain_r.
template <int R>
__device__ __forceinline__ void rng_vector(const RngQueue& q, uint64_t v, uint32_t k0, uint32_t k1, uint32_t thr) {
    const uint64_t ctr = q.base_offset + window_vec(q.win, v) * 32;
    const uint32_t lo = static_cast<uint32_t>(ctr), hi = static_cast<uint32_t>(ctr >> 32);
    uint32_t w0, w1, w2, w3;
    if (lo <= 0xFFFFFFFFu - 31u) {
        w0 = rgo_dev::keep32_nowrap<R>(lo + 0, hi, k0, k1, thr, 0u);
        w1 = rgo_dev::keep32_nowrap<R>(lo + 8, hi, k0, k1, thr, 0u);
        w2 = rgo_dev::keep32_nowrap<R>(lo + 16, hi, k0, k1, thr, 0u);
        w3 = rgo_dev::keep32_nowrap<R>(lo + 24, hi, k0, k1, thr, 0u);
    } else {
        w0 = rgo_dev::keep32<R>(ctr + 0, q.k0, q.k1, q.thr);
        w1 = rgo_dev::keep32<R>(ctr + 8, q.k0, q.k1, q.thr);
        w2 = rgo_dev::keep32<R>(ctr + 16, q.k0, q.k1, q.thr);
        w3 = rgo_dev::keep32<R>(ctr + 24, q.k0, q.k1, q.thr);
    }
    uint8_t* p = q.out + v * 16;
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                 : "memory");
}

// Two vectors at once (independent counters -> interleavable chains).
template <int R>
__device__ __forceinline__ void rng_vector2(const RngQueue& q, uint64_t va, uint64_t vb, uint32_t k0, uint32_t k1,
                                            uint32_t thr) {
    const uint64_t ca = q.base_offset + window_vec(q.win, va) * 32, cb = q.base_offset + window_vec(q.win, vb) * 32;
    const uint32_t la = static_cast<uint32_t>(ca), lb = static_cast<uint32_t>(cb);
    if (la > 0xFFFFFFFFu - 31u || lb > 0xFFFFFFFFu - 31u) {  // rare: a unit straddles a 2^32 counter boundary
        rng_vector<R>(q, va, k0, k1, thr);
        rng_vector<R>(q, vb, k0, k1, thr);
        return;
    }
    const uint32_t ha = static_cast<uint32_t>(ca >> 32), hb = static_cast<uint32_t>(cb >> 32);
    uint32_t wa[4], wb[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        wa[t] = rgo_dev::keep32_nowrap<R>(la + 8 * t, ha, k0, k1, thr, 0u);
        wb[t] = rgo_dev::keep32_nowrap<R>(lb + 8 * t, hb, k0, k1, thr, 0u);
    }
    uint8_t* pa = q.out + va * 16;
    uint8_t* pb = q.out + vb * 16;
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(pa), "r"(wa[0]), "r"(wa[1]), "r"(wa[2]), "r"(wa[3])
                 : "memory");
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(pb), "r"(wb[0]), "r"(wb[1]), "r"(wb[2]), "r"(wb[3])
                 : "memory");
}

// Drain until the queue is empty or (*stop >= stop_at) is observed.
template <int R>
__device__ __forceinline__ void rng_drain_r(const RngQueue& q, const volatile int* stop, int stop_at) {
    const uint32_t lane = threadIdx.x & 31;
    // Keep the key and threshold in vector registers: left to itself the
    // compiler holds them (and the R round keys) in uniform registers, and the
    // RNG's LOP3/compare stream then competes for the uniform datapath that
    // the co-resident GEMM's MMA/TMA warps issue through.
    uint32_t k0 = q.k0, k1 = q.k1, thr = q.thr;
    asm volatile("" : "+r"(k0), "+r"(k1), "+r"(thr) : "r"(lane));
    while (true) {
        if (stop && *stop >= stop_at) break;
        // 64 vectors per claim, two per lane: 16 independent Philox chains
        // per thread keep the fma-heavy pipe fed with few warps
        unsigned long long start = 0;
        if (lane == 0) start = atomicAdd(q.counter, 64ull);
        start = __shfl_sync(0xffffffffu, start, 0);
        if (start >= q.n_vec) break;
        const uint64_t v0 = start + lane, v1 = start + 32 + lane;
        if (v1 < q.n_vec) {
            rng_vector2<R>(q, v0, v1, k0, k1, thr);
        } else {
            if (v0 < q.n_vec) rng_vector<R>(q, v0, k0, k1, thr);
        }
    }
}

// Any round count (runtime loop; slower than the specialisations, same bits).
__device__ __forceinline__ void rng_drain_rt(const RngQueue& q, const volatile int* stop, int stop_at) {
    const uint32_t lane = threadIdx.x & 31;
    while (true) {
        if (stop && *stop >= stop_at) break;
        unsigned long long start = 0;
        if (lane == 0) start = atomicAdd(q.counter, 32ull);
        start = __shfl_sync(0xffffffffu, start, 0);
        if (start >= q.n_vec) break;
        const uint64_t v = start + lane;
        if (v < q.n_vec) {
            const uint64_t ctr = q.base_offset + window_vec(q.win, v) * 32;
            uint32_t w[4];
#pragma unroll 1
            for (int t = 0; t < 4; ++t) w[t] = rgo_dev::keep32_rt(ctr + 8 * t, q.k0, q.k1, q.thr, q.rounds);
            uint8_t* p = q.out + v * 16;
            asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                         "r"(w[3])
                         : "memory");
        }
    }
}

__device__ __forceinline__ void rng_queue_drain(const RngQueue& q, const volatile int* stop, int stop_at = 4) {
    if (q.rounds == 10)
        rng_drain_r<10>(q, stop, stop_at);
    else if (q.rounds == 7)
        rng_drain_r<7>(q, stop, stop_at);
    else if (q.rounds == 5)
        rng_drain_r<5>(q, stop, stop_at);
    else if (q.rounds == 3)
        rng_drain_r<3>(q, stop, stop_at);
    else
        rng_drain_rt(q, stop, stop_at);
}

}  // namespace rgo
