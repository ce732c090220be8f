// attn_bwd_sm100.cu -- K7: Blackwell flash-attention backward with dropout.
//
// The training counterpart of K5/K6 (attn_fwd_sm100.cu).  The reference stops
// at the forward (ref_attention.hpp:56-92; SPEC.md:552 puts backward out of its
// scope), so the semantics are the exact derivative of that forward:
//   P  = softmax(scale * Q K^T) over ALL keys (ref_attention.hpp:78-82)
//   W  = keep ? P / p : 0                     (:84-85, p = float keep_prob)
//   O  = W V
//   dV = W^T dO
//   dP = keep ? (dO V^T) / p : 0
//   D  = rowsum(dO o O)            (= rowsum(P o dP))
//   dS = P o (dP - D)
//   dQ = scale * dS K,   dK = scale * dS^T Q
// with the keep bit of (slice s, query i, key j) = element (s*SQ + i)*SQ + j of
// the reference mask layout (mask.hpp:35-39), read from the bitmask
// (MASK_BITS, the paper's decoupled path) or regenerated with Philox inline
// (MASK_PHILOX, the conventional fused baseline; identical keep decisions).
//
// Three kernels:
//   bwd_prep   per query row: D = dO.O, -lse*log2(e) (padding rows: D 0, -inf),
//              zeroes the fp32 dQ accumulator (HBM-bound, small)
//   bwd_main   one CTA per (slice, 128-key tile); loops over 128-query tiles:
//                S^T  = K Q^T      (SS, TMEM [0,128))
//                dP^T = V dO^T     (SS, TMEM [128,256))
//                dV  += W^T dO     (TS: W^T bf16 from TMEM, dO MN-major)
//                dK  += dS^T Q     (TS: dS^T bf16 from TMEM, Q MN-major)
//                dQ_i = dS K       (SS: dS MN-major from smem, K MN-major) -> TMEM [128,..)
//              keys on TMEM lanes (one thread per key row), so dV/dK
//              accumulate in TMEM for the whole loop; dQ tiles are staged
//              through shared memory and reduced into an fp32 accumulator
//              with TMA bulk reduce-adds (cp.reduce.async.bulk .add.f32).
//   bwd_dq     dQ = scale * accumulator -> bf16
//
// Warp roles of bwd_main (512 threads, 128 registers each):
//   warp 0      TMA: K, V once; Q (+ its -lse2 / D rows) through a 2-stage ring, dO single-buffered
//   warp 1      MMA issuer (one elected lane)
//   warps 4-7   "softmax" WG 0: queries [0,64) of each tile, one thread per key
//   warps 8-11  softmax WG 1: queries [64,128)
//   warps 12-15 dQ drain: TMEM -> smem -> bulk reduce-add into the fp32 accumulator
// Per query tile i the MMA order is  dP(i), dV(i), S(i+1), dK(i), dQ(i):
// the softmax's P phase of tile i overlaps dK(i-1)/dQ(i-1)/dP(i), its dS
// phase overlaps dV(i)/S(i+1).
// Mask bits arrive row-major (16 B per query row per 128-key tile); with keys
// on lanes each warp transposes its 32x32 bit blocks with a 5-stage
// shuffle butterfly.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "attn.h"
#include "philox.cuh"
#include "rgo_internal.h"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace rgo_attn_bwd {

using namespace sm100;
using rgo_attn::MASK_BITS;
using rgo_attn::MASK_NONE;
using rgo_attn::MASK_PHILOX;

constexpr int BQ = 128;   // queries per tile
constexpr int BKV = 128;  // keys per CTA
constexpr int STAGES = 2;     // Q (+ row terms) ring
constexpr int DO_STAGES = 1;  // dO is consumed early in each iteration (dP, dV)
constexpr int THREADS = 512;
constexpr uint32_t TMEM_COLS = 512;
constexpr int MAX_DSMEM = 232448;  // 227 KiB opt-in maximum on sm_100

struct Params {
    int B, H, S, n_qt, n_kt;
    float scale;        // softmax scale (dQ, dK)
    float scale_log2;   // scale * log2(e)
    float inv_keep;     // 1 / float keep_prob (1 without dropout)
    const uint8_t* bits;
    uint64_t bits_bytes;
    int bits_aligned;   // SQ % 32 == 0 and 4-byte aligned bits: one word per row per warp
    uint32_t k0, k1;
    uint64_t base_offset;
    uint32_t thr;
    int rounds;
    const float* rows;  // [slices][n_qt*128][2]: per query tile 128 x -lse*log2e, then 128 x D
    float* dq_acc;      // blocked fp32 accumulator (see dq_index)
    void* dK;
    void* dV;
    long long k_sb, k_sh, k_ss;  // dK strides (elements)
    long long v_sb, v_sh, v_ss;  // dV strides
    int mask_tma;                // v2, MASK_BITS: the keep-bit tile arrives by TMA with Q (SQ % 128 == 0)
    int dkv_tma;                 // v2: dK/dV leave by TMA store (the kernel's tmdK/tmdV)
};

// Blocked dQ accumulator: per (slice, query tile) HD/32 column chunks of 8
// groups x 128 rows x float4 -- the drain's smem staging layout, so each
// 64-column half of a tile is one contiguous 32 KiB bulk reduce.
__host__ __device__ __forceinline__ uint64_t dq_tile_base(uint64_t slice, int n_qt, int qt, int HD) {
    return (slice * n_qt + qt) * static_cast<uint64_t>(BQ) * HD;
}
__host__ __device__ __forceinline__ uint32_t dq_off(int row, int col) {  // within a tile
    return ((static_cast<uint32_t>(col >> 2) * BQ) + row) * 4 + (col & 3);
}

template <int HD>
struct Smem {
    static constexpr int CHUNK = 128 * 128;         // 128 rows x 128 B (one SW128 column block)
    static constexpr int TILE = (HD / 64) * CHUNK;  // 128 rows x HD bf16
    static constexpr int K_OFF = 0;
    static constexpr int V_OFF = TILE;
    static constexpr int Q_OFF = 2 * TILE;
    static constexpr int DO_OFF = Q_OFF + STAGES * TILE;
    static constexpr int DS_OFF = DO_OFF + DO_STAGES * TILE;  // dS [128 keys][128 queries] bf16
    static constexpr int STG_OFF = DS_OFF + 2 * CHUNK;        // dQ staging: 64 columns fp32
    static constexpr int ROW_OFF = STG_OFF + BQ * 64 * 4;     // per stage: 128 -lse2, 128 D
    static constexpr int BAR_OFF = ROW_OFF + STAGES * 1024;
    static constexpr int BYTES = BAR_OFF + 256;
    static constexpr int ALLOC = (BYTES + 1023 <= MAX_DSMEM) ? BYTES + 1023 : MAX_DSMEM;
};

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}

// TMA bulk reduce-add of `bytes` of fp32 from shared memory into global memory
// (performed in L2; no per-lane atomics on the SM).
__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// 32x32 bit transpose across a warp: in, lane l holds row l (bit c = column
// c); out, lane l holds column l (bit r = row r's bit l).  Five butterfly
// stages swap the off-diagonal s x s blocks of lane pairs (l, l^s).
__device__ __forceinline__ uint32_t transpose32(uint32_t a, uint32_t lane) {
    const uint32_t lo_masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int s = 16 >> t;
        const uint32_t lo = lo_masks[t];
        const uint32_t other = __shfl_xor_sync(0xffffffffu, a, s);
        const bool top = (lane & s) == 0;
        const uint32_t x = top ? (other << s) : (other >> s);
        const uint32_t m = top ? lo : ~lo;
        a = (a & m) | (x & ~m);
    }
    return a;
}

// Keep bits of 32 consecutive elements of one query row, starting at global
// element idx0 (bit c = element idx0 + c); elements >= n_valid_cols of the
// row are cleared.
template <int MODE, int R>
__device__ __forceinline__ uint32_t row_word(const Params& p, uint64_t idx0, int n_valid) {
    if (n_valid <= 0) return 0u;
    uint32_t w;
    if constexpr (MODE == MASK_BITS) {
        if (p.bits_aligned) {
            w = __ldg(reinterpret_cast<const uint32_t*>(p.bits) + (idx0 >> 5));
        } else {
            const uint64_t b0 = idx0 >> 3;
            const uint32_t sh = static_cast<uint32_t>(idx0 & 7);
            uint64_t acc = 0;
#pragma unroll
            for (int t = 0; t < 5; ++t) {
                const uint64_t b = b0 + t;
                acc |= static_cast<uint64_t>(b < p.bits_bytes ? p.bits[b] : 0u) << (8 * t);
            }
            w = static_cast<uint32_t>(acc >> sh);
        }
    } else if constexpr (MODE == MASK_PHILOX) {
        if ((idx0 & 3) == 0) {
            const uint64_t ctr = p.base_offset + (idx0 >> 2);
            const uint32_t lo = static_cast<uint32_t>(ctr), hi = static_cast<uint32_t>(ctr >> 32);
            if (R > 0 && lo <= 0xFFFFFFFFu - 7u) {
                w = rgo_dev::keep32_nowrap<(R > 0 ? R : 1)>(lo, hi, p.k0, p.k1, p.thr, 0u);
            } else {
                w = 0;
#pragma unroll 1
                for (int b = 0; b < 8; ++b) {
                    const uint64_t c = ctr + b;
                    const uint4 o = rgo_dev::philox_rt(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32), 0u,
                                                       0u, p.k0, p.k1, p.rounds);
                    w |= (static_cast<uint32_t>(o.x < p.thr) | (static_cast<uint32_t>(o.y < p.thr) << 1) |
                          (static_cast<uint32_t>(o.z < p.thr) << 2) | (static_cast<uint32_t>(o.w < p.thr) << 3))
                         << (4 * b);
                }
            }
        } else {
            w = 0;
#pragma unroll 1
            for (int c = 0; c < 32; ++c) {
                const uint64_t idx = idx0 + c;
                const uint64_t ctr = p.base_offset + (idx >> 2);
                const uint4 o = rgo_dev::philox_rt(static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), 0u,
                                                   0u, p.k0, p.k1, p.rounds);
                const uint32_t ln = static_cast<uint32_t>(idx & 3);
                const uint32_t wd = ln == 0 ? o.x : ln == 1 ? o.y : ln == 2 ? o.z : o.w;
                w |= static_cast<uint32_t>(wd < p.thr) << c;
            }
        }
    } else {
        w = 0xFFFFFFFFu;
    }
    return n_valid >= 32 ? w : (w & ((1u << n_valid) - 1u));
}

__global__ void bwd_prep_kernel(const __nv_bfloat16* __restrict__ O, long long o_sb, long long o_sh, long long o_ss,
                                const __nv_bfloat16* __restrict__ dO, long long d_sb, long long d_sh, long long d_ss,
                                const float* __restrict__ lse, float* __restrict__ rows, float* __restrict__ dq_acc,
                                int B, int H, int S, int n_qt, int HD) {
    const uint64_t padded = static_cast<uint64_t>(n_qt) * BQ;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<uint64_t>(B) * H * padded) return;
    const uint64_t slice = t / padded;
    const int r = static_cast<int>(t - slice * padded);
    const int qt = r / BQ, rr = r % BQ;
    const int bb = static_cast<int>(slice / H), hh = static_cast<int>(slice % H);
    float d = 0.0f, nl = -INFINITY;
    if (r < S) {
        const uint4* po = reinterpret_cast<const uint4*>(O + bb * o_sb + hh * o_sh + static_cast<long long>(r) * o_ss);
        const uint4* pd = reinterpret_cast<const uint4*>(dO + bb * d_sb + hh * d_sh + static_cast<long long>(r) * d_ss);
        float acc0 = 0.0f, acc1 = 0.0f;
        for (int c = 0; c < HD / 8; ++c) {
            const uint4 a = __ldg(po + c), b = __ldg(pd + c);
            const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                acc0 = fmaf(bf16_lo(av[e]), bf16_lo(bv[e]), acc0);
                acc1 = fmaf(bf16_hi(av[e]), bf16_hi(bv[e]), acc1);
            }
        }
        d = acc0 + acc1;
        nl = -lse[slice * S + r] * 1.4426950408889634f;
    }
    float* rw = rows + (slice * n_qt + qt) * (2 * BQ);
    rw[rr] = nl;
    rw[BQ + rr] = d;
    if (!dq_acc) return;  // split backward (v3): dQ accumulates in TMEM, no fp32 accumulator
    float4* acc = reinterpret_cast<float4*>(dq_acc + dq_tile_base(slice, n_qt, qt, HD));
    for (int g = 0; g < HD / 4; ++g) acc[g * BQ + rr] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
}

__global__ void bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dQ, long long q_sb,
                              long long q_sh, long long q_ss, int B, int H, int S, int n_qt, int HD, float scale) {
    // thread = (slice, row, 8-column group): reads 2 float4 (coalesced over
    // rows), writes 16 bytes of bf16
    const int groups = HD / 8;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t padded = static_cast<uint64_t>(n_qt) * BQ;
    const uint64_t per_slice = padded * groups;
    if (t >= static_cast<uint64_t>(B) * H * per_slice) return;
    const uint64_t slice = t / per_slice;
    const uint64_t rem = t - slice * per_slice;
    const int g = static_cast<int>(rem / padded);
    const int r = static_cast<int>(rem - static_cast<uint64_t>(g) * padded);
    if (r >= S) return;
    const int qt = r / BQ, rr = r % BQ;
    const float4* acc = reinterpret_cast<const float4*>(dq_acc + dq_tile_base(slice, n_qt, qt, HD));
    const float4 a = acc[(2 * g) * BQ + rr], b = acc[(2 * g + 1) * BQ + rr];
    const int bb = static_cast<int>(slice / H), hh = static_cast<int>(slice % H);
    uint4 out;
    out.x = pack_bf16(a.x * scale, a.y * scale);
    out.y = pack_bf16(a.z * scale, a.w * scale);
    out.z = pack_bf16(b.x * scale, b.y * scale);
    out.w = pack_bf16(b.z * scale, b.w * scale);
    *reinterpret_cast<uint4*>(dQ + bb * q_sb + hh * q_sh + static_cast<long long>(r) * q_ss + 8 * g) = out;
}

// DQ = false: the dK/dV half of the split backward (launch_attn_bwd3): no dQ
// MMA, no dS staging in shared memory, no drain -- dQ comes from bwd_dq3_kernel.
template <int HD, int MODE, int R, bool DQ>
__global__ void __launch_bounds__(THREADS, 1) bwd_main_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                              const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV,
                                                              const __grid_constant__ CUtensorMap tmdO,
                                                              const Params p) {
    using SM = Smem<HD>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    if (pad + SM::BYTES > static_cast<uint32_t>(SM::ALLOC)) __trap();
    uint8_t* smem = smem_raw + pad;
    uint8_t* sK = smem + SM::K_OFF;
    uint8_t* sV = smem + SM::V_OFF;
    uint8_t* sQ = smem + SM::Q_OFF;
    uint8_t* sdO = smem + SM::DO_OFF;
    uint8_t* sdS = smem + SM::DS_OFF;
    const float* sRows = reinterpret_cast<const float*>(smem + SM::ROW_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;          // [2]
    uint64_t* q_empty = q_full + STAGES;  // [2]
    uint64_t* do_full = q_empty + STAGES;
    uint64_t* do_empty = do_full + DO_STAGES;
    uint64_t* s_full = do_empty + DO_STAGES;
    uint64_t* p_full = s_full + 1;
    uint64_t* dp_full = p_full + 1;
    uint64_t* ds_full = dp_full + 1;
    uint64_t* dq_full = ds_full + 1;
    uint64_t* dq_empty = dq_full + 1;
    uint64_t* acc_full = dq_empty + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int kt = blockIdx.x % p.n_kt;
    const int bh = blockIdx.x / p.n_kt;
    const int hh = bh % p.H, bb = bh / p.H;
    const uint64_t slice = static_cast<uint64_t>(bb) * p.H + hh;
    const int kv0 = kt * BKV;
    const int n_qt = p.n_qt;
    constexpr int NCH = HD / 64;
    // Query tiles are visited starting at the CTA's key-tile index, so the
    // CTAs of one head (which run concurrently) reduce into different dQ tiles.
    auto qtile = [&](int i) { const int t = i + kt % n_qt; return t >= n_qt ? t - n_qt : t; };

    if (warp == 0 && lane == 0) {
        mbar_init(smem_u32(kv_full), 1);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&q_full[s]), 1);
            mbar_init(smem_u32(&q_empty[s]), 1);
        }
        for (int s = 0; s < DO_STAGES; ++s) {
            mbar_init(smem_u32(&do_full[s]), 1);
            mbar_init(smem_u32(&do_empty[s]), 1);
        }
        mbar_init(smem_u32(s_full), 1);
        mbar_init(smem_u32(p_full), 8);
        mbar_init(smem_u32(dp_full), 1);
        mbar_init(smem_u32(ds_full), 8);
        mbar_init(smem_u32(dq_full), 1);
        mbar_init(smem_u32(dq_empty), 4);
        mbar_init(smem_u32(acc_full), 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmdO);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------------------------------ TMA
        if (elect_one()) {
            const uint32_t kb = smem_u32(kv_full);
            mbar_arrive_expect_tx(kb, 2 * SM::TILE);
            for (int c = 0; c < NCH; ++c) {
                tma_load_4d(smem_u32(sK + c * SM::CHUNK), &tmK, kb, c * 64, kv0, hh, bb);
                tma_load_4d(smem_u32(sV + c * SM::CHUNK), &tmV, kb, c * 64, kv0, hh, bb);
            }
        }
        __syncwarp();
        const float* rows = p.rows + slice * n_qt * (2 * BQ);
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            mbar_wait(smem_u32(&q_empty[st]), ph ^ 1);
            if (elect_one()) {
                const uint32_t qb = smem_u32(&q_full[st]);
                mbar_arrive_expect_tx(qb, SM::TILE + 1024);
                for (int c = 0; c < NCH; ++c)
                    tma_load_4d(smem_u32(sQ + st * SM::TILE + c * SM::CHUNK), &tmQ, qb, c * 64, qtile(i) * BQ, hh, bb);
                bulk_load(smem_u32(smem + SM::ROW_OFF + st * 1024), rows + qtile(i) * (2 * BQ), 1024, qb);
            }
            __syncwarp();
            const int dst = i % DO_STAGES;
            mbar_wait(smem_u32(&do_empty[dst]), ((i / DO_STAGES) & 1) ^ 1);
            if (elect_one()) {
                const uint32_t db = smem_u32(&do_full[dst]);
                mbar_arrive_expect_tx(db, SM::TILE);
                for (int c = 0; c < NCH; ++c)
                    tma_load_4d(smem_u32(sdO + dst * SM::TILE + c * SM::CHUNK), &tmdO, db, c * 64, qtile(i) * BQ, hh, bb);
            }
            __syncwarp();
        }
    } else if (warp == 1) {  // ----------------------------------------------------- MMA
        constexpr uint32_t IDESC_T = idesc_make(1, 1, BKV, BQ, 0, 0);   // S^T, dP^T
        constexpr uint32_t IDESC_ACC = idesc_make(1, 1, BKV, HD, 0, 1); // dV, dK (A TMEM, B MN-major)
        constexpr uint32_t IDESC_DQ = idesc_make(1, 1, BQ, HD, 1, 1);   // dQ (A, B MN-major)
        const uint64_t k_kdesc = desc_kmajor_sw128(smem_u32(sK));
        const uint64_t v_kdesc = desc_kmajor_sw128(smem_u32(sV));
        const uint64_t q_kdesc = desc_kmajor_sw128(smem_u32(sQ));
        const uint64_t do_kdesc = desc_kmajor_sw128(smem_u32(sdO));
        const uint64_t q_mdesc = desc_sw128(smem_u32(sQ), SM::CHUNK, 1024);
        const uint64_t do_mdesc = desc_sw128(smem_u32(sdO), SM::CHUNK, 1024);
        const uint64_t k_mdesc = desc_sw128(smem_u32(sK), SM::CHUNK, 1024);
        const uint64_t ds_mdesc = desc_sw128(smem_u32(sdS), SM::CHUNK, 1024);
        const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + HD;
        // D (128 x 128) = A (128 x HD, K-major) . B (128 x HD, K-major)^T
        auto issue_t = [&](uint32_t d, uint64_t a, uint64_t b) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint32_t off = ((kk >> 2) * SM::CHUNK + (kk & 3) * 32) >> 4;
                mma_f16_ss(d, a + off, b + off, IDESC_T, kk > 0);
            }
        };
        // D (128 keys x HD) += A^T from TMEM (bf16 pairs: queries 64h+16m.. at
        // column 64h + 8m) . B (128 queries x HD, MN-major)
        auto issue_acc = [&](uint32_t d, uint32_t a_tmem, uint64_t b, bool acc) {
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk)
                mma_f16_ts(d, a_tmem + (kk >> 2) * 64 + (kk & 3) * 8, b + ((kk * 2048) >> 4), IDESC_ACC,
                           (acc || kk > 0) ? 1u : 0u);
        };
        mbar_wait(smem_u32(kv_full), 0);
        mbar_wait(smem_u32(&q_full[0]), 0);
        tc_fence_after();
        if (elect_one()) {
            issue_t(tS, k_kdesc, q_kdesc);
            tc_commit(smem_u32(s_full));
        }
        __syncwarp();
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const uint32_t soff = (st * SM::TILE) >> 4;
            const int dst = i % DO_STAGES;
            const uint32_t doff = (dst * SM::TILE) >> 4;
            mbar_wait(smem_u32(&do_full[dst]), (i / DO_STAGES) & 1);
            if (DQ && i > 0) mbar_wait(smem_u32(dq_empty), (i - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_t(tdP, v_kdesc, do_kdesc + doff);
                tc_commit(smem_u32(dp_full));
            }
            __syncwarp();
            mbar_wait(smem_u32(p_full), i & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_acc(tdV, tS, do_mdesc + doff, i > 0);
                tc_commit(smem_u32(&do_empty[dst]));
            }
            __syncwarp();
            if (i + 1 < n_qt) {
                const int st1 = (i + 1) & 1;
                mbar_wait(smem_u32(&q_full[st1]), ((i + 1) >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    issue_t(tS, k_kdesc, q_kdesc + ((st1 * SM::TILE) >> 4));
                    tc_commit(smem_u32(s_full));
                }
                __syncwarp();
            }
            mbar_wait(smem_u32(ds_full), i & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_acc(tdK, tdP, q_mdesc + soff, i > 0);
                if constexpr (DQ) {
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk)
                        mma_f16_ss(tdP, ds_mdesc + ((kk * 2048) >> 4), k_mdesc + ((kk * 2048) >> 4), IDESC_DQ,
                                   kk > 0);
                }
                tc_commit(smem_u32(&q_empty[st]));
                if constexpr (DQ) tc_commit(smem_u32(dq_full));
                if (i + 1 == n_qt) tc_commit(smem_u32(acc_full));
            }
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 12) {  // --------------------------------- softmax / dS
        const int h = (warp - 4) >> 2;         // query half of each tile
        const uint32_t qw = warp & 3;          // TMEM lane quarter
        const int r = static_cast<int>(qw * 32 + lane);  // key row within the CTA tile
        const bool key_valid = kv0 + r < p.S;
        const uint32_t lane_base = (qw * 32) << 16;
        const uint32_t tS = tmem + lane_base + 64 * h;
        const uint32_t tdP = tmem + lane_base + 128 + 64 * h;
        const int kcol = kv0 + static_cast<int>(qw) * 32;  // first key of this warp's 32
        const int kvalid = p.S - kcol;                     // valid keys in the warp's word
        uint8_t* ds_row = sdS + h * SM::CHUNK + r * 128;
        const uint32_t sw = static_cast<uint32_t>(r & 7);
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            // keep words: bit e of kw[c] = keep(query i*128 + 64h + 32c + e, key kv0 + r)
            uint32_t kw[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int qrow = qtile(i) * BQ + 64 * h + 32 * c + static_cast<int>(lane);
                uint32_t w = 0;
                if (qrow < p.S) w = row_word<MODE, R>(p, (slice * p.S + qrow) * static_cast<uint64_t>(p.S) + kcol, kvalid);
                kw[c] = transpose32(w, lane);
            }
            if (!key_valid) kw[0] = kw[1] = 0;
            const float* nlse = sRows + st * 256 + 64 * h;
            const float* Dv = nlse + BQ;
            mbar_wait(smem_u32(&q_full[st]), ph);  // rows of tile i landed (already complete)
            mbar_wait(smem_u32(s_full), i & 1);
            tc_fence_after();
            // ---- P phase: P = 2^(s*scale*log2e - lse*log2e); W = keep ? P : 0 -> TMEM (bf16)
            uint32_t pb[2][16];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t s[32];
                tmem_ld32(tS + 32 * c, s);
                tmem_ld_wait_regs(s);
                uint32_t wpk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    const float4 nl = *reinterpret_cast<const float4*>(nlse + 32 * c + e);
                    const float2 t0 = __ffma2_rn(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sc2,
                                                 make_float2(nl.x, nl.y));
                    const float2 t1 = __ffma2_rn(make_float2(__uint_as_float(s[e + 2]), __uint_as_float(s[e + 3])),
                                                 sc2, make_float2(nl.z, nl.w));
                    const float p0 = ex2_approx(t0.x), p1 = ex2_approx(t0.y);
                    const float p2 = ex2_approx(t1.x), p3 = ex2_approx(t1.y);
                    pb[c][e / 2] = pack_bf16(p0, p1);
                    pb[c][e / 2 + 1] = pack_bf16(p2, p3);
                    wpk[e / 2] = pack_bf16(((kw[c] >> e) & 1u) ? p0 : 0.0f, ((kw[c] >> (e + 1)) & 1u) ? p1 : 0.0f);
                    wpk[e / 2 + 1] =
                        pack_bf16(((kw[c] >> (e + 2)) & 1u) ? p2 : 0.0f, ((kw[c] >> (e + 3)) & 1u) ? p3 : 0.0f);
                }
                tmem_st16(tS + 16 * c, wpk);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(p_full));
            // ---- dS phase: dS = P o (keep ? dP/p : 0 - D) -> TMEM (bf16, for dK) and smem (for dQ)
            mbar_wait(smem_u32(dp_full), i & 1);
                    tc_fence_after();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t d[32];
                tmem_ld32(tdP + 32 * c, d);
                tmem_ld_wait_regs(d);
                uint32_t dpk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    const float4 dd = *reinterpret_cast<const float4*>(Dv + 32 * c + e);
                    const float dv[4] = {dd.x, dd.y, dd.z, dd.w};
                    float ds[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t pw = pb[c][(e + u) / 2];
                        const float pv = ((e + u) & 1) ? bf16_hi(pw) : bf16_lo(pw);
                        const float dp = ((kw[c] >> (e + u)) & 1u) ? __uint_as_float(d[e + u]) * p.inv_keep : 0.0f;
                        ds[u] = pv * (dp - dv[u]);
                    }
                    dpk[e / 2] = pack_bf16(ds[0], ds[1]);
                    dpk[e / 2 + 1] = pack_bf16(ds[2], ds[3]);
                }
                tmem_st16(tdP + 16 * c, dpk);
                if constexpr (DQ) {
                    // smem dS row (key r), queries 64h + 32c.. : 16-byte units 4c..4c+3 of line r
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t unit = (4 * c + u) ^ sw;
                        *reinterpret_cast<uint4*>(ds_row + unit * 16) =
                            make_uint4(dpk[4 * u], dpk[4 * u + 1], dpk[4 * u + 2], dpk[4 * u + 3]);
                    }
                }
            }
            if constexpr (DQ) fence_proxy_async_smem();
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(ds_full));
        }
        // ---- epilogue: dV = acc / keep_prob, dK = acc * scale; columns [h*HD/2, (h+1)*HD/2)
        mbar_wait(smem_u32(acc_full), 0);
        tc_fence_after();
        const int key = kv0 + r;
        __nv_bfloat16* dv_row = static_cast<__nv_bfloat16*>(p.dV) + bb * p.v_sb + hh * p.v_sh +
                                static_cast<long long>(key_valid ? key : 0) * p.v_ss;
        __nv_bfloat16* dk_row = static_cast<__nv_bfloat16*>(p.dK) + bb * p.k_sb + hh * p.k_sh +
                                static_cast<long long>(key_valid ? key : 0) * p.k_ss;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {
            const uint32_t tacc = tmem + lane_base + 256 + which * HD;
            const float mul = which == 0 ? p.inv_keep : p.scale;
            __nv_bfloat16* dst = which == 0 ? dv_row : dk_row;
#pragma unroll 1
            for (int c = 0; c < HD / 64; ++c) {
                const int col = h * (HD / 2) + 32 * c;
                uint32_t o[32];
                tmem_ld32(tacc + col, o);
                tmem_ld_wait_regs(o);
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    pk[e] = pack_bf16(__uint_as_float(o[2 * e]) * mul, __uint_as_float(o[2 * e + 1]) * mul);
                if (key_valid) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
                    for (int v = 0; v < 4; ++v) d4[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                }
            }
        }
    } else if (DQ && warp >= 12) {  // ------------------------------------------- dQ drain
        // TMEM -> smem staging (64 columns, the accumulator's blocked layout)
        // -> one 32 KiB TMA bulk reduce-add per half.  The second half is held
        // in registers while the first is staged, so TMEM is released before
        // the staging buffer has to be reused.
        const uint32_t qw = warp & 3;
        const int r = static_cast<int>(qw * 32 + lane);
        const uint32_t tdq = tmem + ((qw * 32) << 16) + 128;
        float4* stg = reinterpret_cast<float4*>(smem + SM::STG_OFF);
        const uint32_t stg_addr = smem_u32(stg);
        const bool leader = warp == 12 && lane == 0;
        constexpr uint32_t HALF_BYTES = BQ * 64 * 4;
        auto stage = [&](const uint32_t (&v)[32], int c_local) {
#pragma unroll
            for (int g = 0; g < 8; ++g)
                stg[(c_local * 8 + g) * BQ + r] = make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                                             __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3]));
        };
        auto flush = [&](float* gdst) {  // all 4 drain warps staged -> one bulk reduce
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (leader) {
                bulk_reduce_add_f32(gdst, stg_addr, HALF_BYTES);
                bulk_commit();
            }
        };
        auto staging_free = [&]() {
            if (leader) bulk_wait_read0();
            named_bar_sync(1, 128);
        };
        for (int i = 0; i < n_qt; ++i) {
            mbar_wait(smem_u32(dq_full), i & 1);
            tc_fence_after();
            float* acc = p.dq_acc + dq_tile_base(slice, n_qt, qtile(i), HD);
            uint32_t hi0[32], hi1[32];
            staging_free();
            {
                uint32_t v[32];
                tmem_ld32(tdq, v);
                tmem_ld_wait_regs(v);
                stage(v, 0);
                tmem_ld32(tdq + 32, v);
                tmem_ld_wait_regs(v);
                stage(v, 1);
            }
            if constexpr (HD == 128) {
                tmem_ld32(tdq + 64, hi0);
                tmem_ld32(tdq + 96, hi1);
                tmem_ld_wait();
                reg_fence(hi0);
                reg_fence(hi1);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(dq_empty));  // TMEM dQ region free
            flush(acc);
            if constexpr (HD == 128) {
                staging_free();
                stage(hi0, 0);
                stage(hi1, 1);
                flush(acc + BQ * 64);
            }
        }
        if (leader) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// ============================================================================
// K7 for head_dim 128 with 64-query tiles ("v2").  Same math and warp roles as
// bwd_main_kernel; the smaller query tile halves the TMEM the scores need, which
// leaves room for a double-buffered dQ^T accumulator, so the tensor core never
// waits for the dQ drain:
//   TMEM  S^T [0,64)  dP^T [64,128)  dQ^T x2 [128,256)  dV [256,384)  dK [384,512)
//   S^T  = K Q^T   (M 128 keys, N 64)      dP^T = V dO^T
//   dV  += W^T dO  (TS, K = 64 queries)    dK  += dS^T Q
//   dQ^T = K^T dS^T (M 128 = head dims, N 64 queries, K 128 keys; both operands
//          MN-major from smem), drained TMEM -> smem -> 32 KiB TMA bulk
//          reduce-add, double-buffered staging.
//
// K^T in TMEM (RGO_BWD_KT_TMEM, default on): the dQ^T MMA reads its A operand,
// K^T, from TMEM (TS mode) instead of re-reading the 32 KB K tile from shared
// memory for every query tile -- the kernel is bound by shared-memory
// bandwidth (ncu: tensor-core operand reads 56 % + LSU 33 % of the SM's smem
// wavefronts), and this removes 256 of the 1408 tensor-core wavefronts per
// tile.  The 64 columns come from the dQ^T double buffer, which single
// buffering does not need (the drain copies dQ^T(i) out of TMEM right after
// it completes, a full tile before dQ^T(i+1) is issued).  The dQ-drain warps
// build K^T once per CTA (thread = head dim, 128 keys -> 64 bf16x2 columns):
//   TMEM  S^T [0,64)  dP^T [64,128)  dQ^T [128,192)  K^T [192,256)  dV  dK
// ============================================================================
constexpr int BQ2 = 64;
#ifndef RGO_BWD_KT_TMEM
#define RGO_BWD_KT_TMEM 1
#endif
constexpr bool KT_TMEM = RGO_BWD_KT_TMEM != 0;
constexpr int DQ_BUFS = KT_TMEM ? 1 : 2;  // dQ^T accumulators in TMEM
// Keep-bit tiles (MASK_BITS, TMA) travel in their own ring, released by the
// softmax warps as soon as they hold their words: each tile is 64 rows x 16
// bytes, SQ/8 bytes apart, and loaded with the Q tile (on q_full) its latency
// gated the Q ring and with it the tensor core.  Measured at B4 H32 S4096
// (profiles/r02_bwd_experiments.md): bits 2.98-3.09 -> 2.92-2.95 ms with 2
// stages; 3/4/8 stages 2.95-3.05 ms; per-lane 4-byte loads 2-4 tiles ahead
// instead of TMA 3.35-3.51 ms.
#ifndef RGO_BWD_MSK_STAGES
#define RGO_BWD_MSK_STAGES 2
#endif
constexpr int MSK_STAGES = RGO_BWD_MSK_STAGES;
// Each ring slot holds the keep bits of two consecutive query tiles (one 128-row TMA box;
// tiles 2u and 2u+1 of the rotated order are always adjacent: the rotation is even).
constexpr int MSK_SLOT = 2 * 1024;
#ifndef RGO_BWD_DKV_TMA
#define RGO_BWD_DKV_TMA 1
#endif

struct Smem2 {
    static constexpr int KCHUNK = 128 * 128;  // K/V: 128 rows x 128 B per 64-dim chunk
    static constexpr int QCHUNK = 64 * 128;   // Q/dO: 64 rows x 128 B
    static constexpr int KTILE = 2 * KCHUNK;
    static constexpr int QTILE = 2 * QCHUNK;
    static constexpr int K_OFF = 0;
    static constexpr int V_OFF = KTILE;
    static constexpr int Q_OFF = 2 * KTILE;
    static constexpr int DO_OFF = Q_OFF + 2 * QTILE;
    static constexpr int DS_OFF = DO_OFF + 2 * QTILE;       // dS [128 keys][64 queries] bf16
    static constexpr int STG_OFF = DS_OFF + 128 * 128;      // 2 x dQ^T tile (128 x 64 fp32)
    static constexpr int STG_BYTES = 128 * BQ2 * 4;
    static constexpr int ROW_OFF = STG_OFF + 2 * STG_BYTES; // per stage: 64 -lse2, 64 D
    static constexpr int MSK_OFF = ROW_OFF + 2 * 512;        // per stage: 64 query rows x 16 B of keep bits
    static constexpr int BAR_OFF = MSK_OFF + MSK_STAGES * MSK_SLOT;
    static constexpr int BYTES = BAR_OFF + 512;
    static constexpr int ALLOC = BYTES + 1023;
};

__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

// Accumulator of one (slice, 64-query tile): [16 query groups][128 dims][4 queries].
__host__ __device__ __forceinline__ uint64_t dq2_tile_base(uint64_t slice, int n_qt, int qt) {
    return (slice * n_qt + qt) * static_cast<uint64_t>(BQ2) * 128;
}

// Row terms of the 64-query-tile backward: D = dO . O and -lse*log2(e) per query row
// (padding rows: 0, -inf).  Sixteen threads per row, each reading 16 bytes of O and dO,
// so a warp reads two whole 256-byte rows per instruction; the fp32 dQ accumulator
// (dq_zero float4s) is zeroed by the same grid, coalesced, instead of a separate memset.
__global__ void bwd_prep2_kernel(const __nv_bfloat16* __restrict__ O, long long o_sb, long long o_sh, long long o_ss,
                                 const __nv_bfloat16* __restrict__ dO, long long d_sb, long long d_sh, long long d_ss,
                                 const float* __restrict__ lse, float* __restrict__ rows, int B, int H, int S,
                                 int n_qt, float4* __restrict__ dq_zero, uint64_t n_zero) {
    const uint64_t padded = static_cast<uint64_t>(n_qt) * BQ2;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n_thr = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t z = t; z < n_zero; z += n_thr) dq_zero[z] = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint64_t row = t >> 4;
    const int part = static_cast<int>(t & 15);
    // rows is a multiple of 64, so only whole warps of the last block exit here and the
    // 16-lane shuffles below always run with full warps
    if (row >= static_cast<uint64_t>(B) * H * padded) return;
    const uint64_t slice = row / padded;
    const int r = static_cast<int>(row - slice * padded);
    const int qt = r / BQ2, rr = r % BQ2;
    const int bb = static_cast<int>(slice / H), hh = static_cast<int>(slice % H);
    float d = 0.0f;
    if (r < S) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(O + bb * o_sb + hh * o_sh + static_cast<long long>(r) * o_ss) + part);
        const uint4 c = __ldg(reinterpret_cast<const uint4*>(dO + bb * d_sb + hh * d_sh + static_cast<long long>(r) * d_ss) + part);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) d = fmaf(bf16_hi(av[e]), bf16_hi(cv[e]), fmaf(bf16_lo(av[e]), bf16_lo(cv[e]), d));
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
    if (part == 0) {
        float* rw = rows + (slice * n_qt + qt) * (2 * BQ2);
        rw[rr] = r < S ? -lse[slice * S + r] * 1.4426950408889634f : -INFINITY;
        rw[BQ2 + rr] = d;
    }
}

// dQ = scale * accumulator -> bf16 rows.  One 256-thread block per (slice, 64-query tile):
// the tile's blocked accumulator ([16 query groups][128 dims][4 queries] fp32, 32 KB) is read
// with 512-byte coalesced float4 loads into shared memory (one float4 of padding every 8, so
// the transposing reads below are conflict-free), then thread (query group, 8 dims) converts
// its 4 x 8 values and writes 4 rows x 16 bytes (a half-warp writes whole 256-byte rows).
__global__ void __launch_bounds__(256) bwd_dq2_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dQ,
                                                      long long q_sb, long long q_sh, long long q_ss, int B, int H, int S,
                                                      int n_qt, float scale) {
    constexpr int N4 = BQ2 * 128 / 4;  // 2048 float4
    __shared__ float4 tile_s[N4 + N4 / 8];
    const uint64_t tile = blockIdx.x;  // slice * n_qt + qt
    const float4* acc = reinterpret_cast<const float4*>(dq_acc + tile * BQ2 * 128);
#pragma unroll
    for (int k = 0; k < N4 / 256; ++k) {
        const int i = threadIdx.x + 256 * k;
        tile_s[i + (i >> 3)] = acc[i];
    }
    __syncthreads();
    const uint64_t slice = tile / n_qt;
    const int qt = static_cast<int>(tile - slice * n_qt);
    const int bb = static_cast<int>(slice / H), hh = static_cast<int>(slice % H);
    const int dg = threadIdx.x & 15, qg = threadIdx.x >> 4;
    float4 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int i = qg * 128 + dg * 8 + e;
        v[e] = tile_s[i + (i >> 3)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int q = qt * BQ2 + qg * 4 + u;
        if (q >= S) break;
        float x[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = (u == 0 ? v[e].x : u == 1 ? v[e].y : u == 2 ? v[e].z : v[e].w) * scale;
        uint4 o;
        o.x = pack_bf16(x[0], x[1]);
        o.y = pack_bf16(x[2], x[3]);
        o.z = pack_bf16(x[4], x[5]);
        o.w = pack_bf16(x[6], x[7]);
        *reinterpret_cast<uint4*>(dQ + bb * q_sb + hh * q_sh + static_cast<long long>(q) * q_ss + dg * 8) = o;
    }
}

template <int MODE, int R>
__global__ void __launch_bounds__(THREADS, 1) bwd_main2_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                               const __grid_constant__ CUtensorMap tmK,
                                                               const __grid_constant__ CUtensorMap tmV,
                                                               const __grid_constant__ CUtensorMap tmdO,
                                                               const __grid_constant__ CUtensorMap tmM,
                                                               const __grid_constant__ CUtensorMap tmdK,
                                                               const __grid_constant__ CUtensorMap tmdV,
                                                               const Params p) {
    using SM = Smem2;
    constexpr int HD = 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* sK = smem + SM::K_OFF;
    uint8_t* sV = smem + SM::V_OFF;
    uint8_t* sQ = smem + SM::Q_OFF;
    uint8_t* sdO = smem + SM::DO_OFF;
    uint8_t* sdS = smem + SM::DS_OFF;
    const float* sRows = reinterpret_cast<const float*>(smem + SM::ROW_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    uint64_t* kv_full = bars;
    uint64_t* q_full = bars + 1;     // [2]
    uint64_t* q_empty = q_full + 2;  // [2]
    uint64_t* do_full = q_empty + 2; // [2]
    uint64_t* do_empty = do_full + 2;
    uint64_t* s_full = do_empty + 2;
    uint64_t* p_full = s_full + 1;
    uint64_t* dp_full = p_full + 1;
    uint64_t* ds_full = dp_full + 1;
    uint64_t* dq_full = ds_full + 1;   // [2]
    uint64_t* dq_empty = dq_full + 2;  // [2]
    uint64_t* acc_full = dq_empty + 2;
    uint64_t* kt_full = acc_full + 1;  // K^T in TMEM (KT_TMEM)
    uint64_t* m_full = kt_full + 1;    // [MSK_STAGES] keep-bit tiles (MASK_BITS, TMA)
    uint64_t* m_empty = m_full + MSK_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(m_empty + MSK_STAGES);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int kt = blockIdx.x % p.n_kt;
    const int bh = blockIdx.x / p.n_kt;
    const int hh = bh % p.H, bb = bh / p.H;
    const uint64_t slice = static_cast<uint64_t>(bb) * p.H + hh;
    const int kv0 = kt * BKV;
    const int n_qt = p.n_qt;  // 64-query tiles
    auto qtile = [&](int i) { const int t = i + (2 * kt) % n_qt; return t >= n_qt ? t - n_qt : t; };

    if (warp == 0 && lane == 0) {
        mbar_init(smem_u32(kv_full), 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&q_full[s]), 1);
            mbar_init(smem_u32(&q_empty[s]), 1);
            mbar_init(smem_u32(&do_full[s]), 1);
            mbar_init(smem_u32(&do_empty[s]), 1);
            mbar_init(smem_u32(&dq_full[s]), 1);
            mbar_init(smem_u32(&dq_empty[s]), 4);
        }
        mbar_init(smem_u32(s_full), 1);
        mbar_init(smem_u32(p_full), 8);
        mbar_init(smem_u32(dp_full), 1);
        mbar_init(smem_u32(ds_full), 8);
        mbar_init(smem_u32(acc_full), 1);
        mbar_init(smem_u32(kt_full), 4);
        for (int s = 0; s < MSK_STAGES; ++s) {
            mbar_init(smem_u32(&m_full[s]), 1);
            mbar_init(smem_u32(&m_empty[s]), 8);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmdO);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------------------------------ TMA
        if (elect_one()) {
            const uint32_t kb = smem_u32(kv_full);
            mbar_arrive_expect_tx(kb, 2 * SM::KTILE);
            for (int c = 0; c < 2; ++c) {
                tma_load_4d(smem_u32(sK + c * SM::KCHUNK), &tmK, kb, c * 64, kv0, hh, bb);
                tma_load_4d(smem_u32(sV + c * SM::KCHUNK), &tmV, kb, c * 64, kv0, hh, bb);
            }
        }
        __syncwarp();
        const float* rows = p.rows + slice * n_qt * (2 * BQ2);
        const bool mtma = MODE == MASK_BITS && p.mask_tma;
        // keep bits of (128 query rows of tiles 2u, 2u+1) x (this CTA's 128 keys) into slot u % MSK_STAGES
        const int n_pairs_q = n_qt / 2;  // mask_tma implies SQ % 128 == 0: n_qt even
        auto load_mask = [&](int u) {
            const int ms = u % MSK_STAGES;
            mbar_wait(smem_u32(&m_empty[ms]), ((u / MSK_STAGES) & 1) ^ 1);
            if (elect_one()) {
                const uint32_t mb = smem_u32(&m_full[ms]);
                mbar_arrive_expect_tx(mb, MSK_SLOT);
                tma_load_2d(smem_u32(smem + SM::MSK_OFF + ms * MSK_SLOT), &tmM, mb, kv0 / 8,
                            static_cast<int>(slice) * p.S + qtile(2 * u) * BQ2);
            }
            __syncwarp();
        };
        if (mtma)
            for (int u = 0; u < MSK_STAGES - 1 && u < n_pairs_q; ++u) load_mask(u);
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int qt = qtile(i);
            mbar_wait(smem_u32(&q_empty[st]), ph ^ 1);
            if (elect_one()) {
                const uint32_t qb = smem_u32(&q_full[st]);
                mbar_arrive_expect_tx(qb, SM::QTILE + 512);
                for (int c = 0; c < 2; ++c)
                    tma_load_4d(smem_u32(sQ + st * SM::QTILE + c * SM::QCHUNK), &tmQ, qb, c * 64, qt * BQ2, hh, bb);
                bulk_load(smem_u32(smem + SM::ROW_OFF + st * 512), rows + qt * (2 * BQ2), 512, qb);
            }
            __syncwarp();
            if (mtma && !(i & 1) && i / 2 + MSK_STAGES - 1 < n_pairs_q) load_mask(i / 2 + MSK_STAGES - 1);
            mbar_wait(smem_u32(&do_empty[st]), ph ^ 1);
            if (elect_one()) {
                const uint32_t db = smem_u32(&do_full[st]);
                mbar_arrive_expect_tx(db, SM::QTILE);
                for (int c = 0; c < 2; ++c)
                    tma_load_4d(smem_u32(sdO + st * SM::QTILE + c * SM::QCHUNK), &tmdO, db, c * 64, qt * BQ2, hh, bb);
            }
            __syncwarp();
        }
    } else if (warp == 1) {  // ----------------------------------------------------- MMA
        constexpr uint32_t IDESC_T = idesc_make(1, 1, BKV, BQ2, 0, 0);  // S^T, dP^T
        constexpr uint32_t IDESC_ACC = idesc_make(1, 1, BKV, HD, 0, 1); // dV, dK
        // dQ^T: A = K^T MN-major from smem, or (KT_TMEM) from TMEM
        constexpr uint32_t IDESC_DQ = idesc_make(1, 1, HD, BQ2, KT_TMEM ? 0 : 1, 1);
        const uint64_t k_kdesc = desc_kmajor_sw128(smem_u32(sK));
        const uint64_t v_kdesc = desc_kmajor_sw128(smem_u32(sV));
        const uint64_t q_kdesc = desc_kmajor_sw128(smem_u32(sQ));
        const uint64_t do_kdesc = desc_kmajor_sw128(smem_u32(sdO));
        const uint64_t q_mdesc = desc_sw128(smem_u32(sQ), SM::QCHUNK, 1024);
        const uint64_t do_mdesc = desc_sw128(smem_u32(sdO), SM::QCHUNK, 1024);
        const uint64_t k_mdesc = desc_sw128(smem_u32(sK), SM::KCHUNK, 1024);
        const uint64_t ds_mdesc = desc_sw128(smem_u32(sdS), SM::KCHUNK, 1024);
        const uint32_t tS = tmem, tdP = tmem + 64, tdV = tmem + 256, tdK = tmem + 384;
        auto issue_t = [&](uint32_t d, uint64_t a, uint64_t b) {  // 128 x 64 x HD, K-major A and B
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint32_t aoff = ((kk >> 2) * SM::KCHUNK + (kk & 3) * 32) >> 4;
                const uint32_t boff = ((kk >> 2) * SM::QCHUNK + (kk & 3) * 32) >> 4;
                mma_f16_ss(d, a + aoff, b + boff, IDESC_T, kk > 0);
            }
        };
        auto issue_acc = [&](uint32_t d, uint32_t a_tmem, uint64_t b, bool acc) {  // K = 64 queries
#pragma unroll
            for (int kk = 0; kk < BQ2 / 16; ++kk)
                mma_f16_ts(d, a_tmem + (kk >> 1) * 32 + (kk & 1) * 8, b + ((kk * 2048) >> 4), IDESC_ACC,
                           (acc || kk > 0) ? 1u : 0u);
        };
        mbar_wait(smem_u32(kv_full), 0);
        mbar_wait(smem_u32(&q_full[0]), 0);
        tc_fence_after();
        if (elect_one()) {
            issue_t(tS, k_kdesc, q_kdesc);
            tc_commit(smem_u32(s_full));
        }
        __syncwarp();
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const uint32_t soff = (st * SM::QTILE) >> 4;
            mbar_wait(smem_u32(&do_full[st]), ph);
            tc_fence_after();
            if (elect_one()) {
                issue_t(tdP, v_kdesc, do_kdesc + soff);
                tc_commit(smem_u32(dp_full));
            }
            __syncwarp();
            mbar_wait(smem_u32(p_full), i & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_acc(tdV, tS, do_mdesc + soff, i > 0);
                tc_commit(smem_u32(&do_empty[st]));
            }
            __syncwarp();
            if (i + 1 < n_qt) {
                const int st1 = st ^ 1;
                mbar_wait(smem_u32(&q_full[st1]), ((i + 1) >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    issue_t(tS, k_kdesc, q_kdesc + ((st1 * SM::QTILE) >> 4));
                    tc_commit(smem_u32(s_full));
                }
                __syncwarp();
            }
            mbar_wait(smem_u32(ds_full), i & 1);
            const int b = DQ_BUFS == 2 ? (i & 1) : 0;
            if (i >= DQ_BUFS) mbar_wait(smem_u32(&dq_empty[b]), ((i / DQ_BUFS) - 1) & 1);
            if (KT_TMEM && i == 0) mbar_wait(smem_u32(kt_full), 0);
            tc_fence_after();
            if (elect_one()) {
                issue_acc(tdK, tdP, q_mdesc + soff, i > 0);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    if constexpr (KT_TMEM)
                        mma_f16_ts(tmem + 128, tmem + 192 + kk * 8, ds_mdesc + ((kk * 2048) >> 4), IDESC_DQ, kk > 0);
                    else
                        mma_f16_ss(tmem + 128 + 64 * b, k_mdesc + ((kk * 2048) >> 4), ds_mdesc + ((kk * 2048) >> 4),
                                   IDESC_DQ, kk > 0);
                }
                tc_commit(smem_u32(&q_empty[st]));
                tc_commit(smem_u32(&dq_full[b]));
                if (i + 1 == n_qt) tc_commit(smem_u32(acc_full));
            }
            __syncwarp();
        }
    } else if (warp >= 4 && warp < 12) {  // --------------------------------- softmax / dS
        const int h = (warp - 4) >> 2;         // 32-query half of each 64-query tile
        const uint32_t qw = warp & 3;
        const int r = static_cast<int>(qw * 32 + lane);  // key row
        const bool key_valid = kv0 + r < p.S;
        const uint32_t lane_base = (qw * 32) << 16;
        const uint32_t tS = tmem + lane_base + 32 * h;
        const uint32_t tdP = tmem + lane_base + 64 + 32 * h;
        const int kcol = kv0 + static_cast<int>(qw) * 32;
        const int kvalid = p.S - kcol;
        uint8_t* ds_row = sdS + r * 128;
        const uint32_t sw = static_cast<uint32_t>(r & 7);
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        for (int i = 0; i < n_qt; ++i) {
            const int st = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int qrow = qtile(i) * BQ2 + 32 * h + static_cast<int>(lane);
            const float* nlse = sRows + st * 128 + 32 * h;
            const float* Dv = nlse + BQ2;
#if defined(RGO_BWD_DIAG) && (RGO_BWD_DIAG & 1)  // timing diagnostic: no softmax/dS work
            if (MODE == MASK_BITS && p.mask_tma) {
                mbar_wait(smem_u32(&m_full[(i / 2) % MSK_STAGES]), ((i / 2) / MSK_STAGES) & 1);
                __syncwarp();
                if (lane == 0 && (i & 1)) mbar_arrive(smem_u32(&m_empty[(i / 2) % MSK_STAGES]));
            }
            mbar_wait(smem_u32(&q_full[st]), ph);
            mbar_wait(smem_u32(s_full), i & 1);
            tc_fence_after();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(p_full));
            mbar_wait(smem_u32(dp_full), i & 1);
            tc_fence_after();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(ds_full));
            if (true) continue;
#endif
            uint32_t w = 0;
            if (MODE == MASK_BITS && p.mask_tma) {  // this lane's query row, this warp's 32 keys, from smem
                const int ms = (i / 2) % MSK_STAGES;
                mbar_wait(smem_u32(&m_full[ms]), ((i / 2) / MSK_STAGES) & 1);
                w = reinterpret_cast<const uint32_t*>(smem + SM::MSK_OFF + ms * MSK_SLOT)
                    [((i & 1) * BQ2 + 32 * h + lane) * 4 + qw];
                __syncwarp();
                if (lane == 0 && (i & 1)) mbar_arrive(smem_u32(&m_empty[ms]));  // both tiles' words read
                mbar_wait(smem_u32(&q_full[st]), ph);  // row terms of tile i landed
            } else {
                if (qrow < p.S)
                    w = row_word<MODE, R>(p, (slice * p.S + qrow) * static_cast<uint64_t>(p.S) + kcol, kvalid);
                mbar_wait(smem_u32(&q_full[st]), ph);  // row terms of tile i landed
            }
            uint32_t kw = transpose32(w, lane);  // bit e: keep(query tile*64 + 32h + e, key kv0 + r)
            if (!key_valid) kw = 0;
            mbar_wait(smem_u32(s_full), i & 1);
            tc_fence_after();
            uint32_t pb[16];
            {
                uint32_t s[32];
                tmem_ld32(tS, s);
                tmem_ld_wait_regs(s);
                uint32_t ksh[8];  // W^T = P with dropped pairs' halves cleared (keep_pair_mask, attn.h)
#pragma unroll
                for (int t = 0; t < 8; ++t) ksh[t] = kw << t;
                uint32_t wpk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    const float4 nl = *reinterpret_cast<const float4*>(nlse + e);
                    const float2 t0 = __ffma2_rn(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sc2,
                                                 make_float2(nl.x, nl.y));
                    const float2 t1 = __ffma2_rn(make_float2(__uint_as_float(s[e + 2]), __uint_as_float(s[e + 3])),
                                                 sc2, make_float2(nl.z, nl.w));
                    const float p0 = ex2_approx(t0.x), p1 = ex2_approx(t0.y);
                    const float p2 = ex2_approx(t1.x), p3 = ex2_approx(t1.y);
                    pb[e / 2] = pack_bf16(p0, p1);
                    pb[e / 2 + 1] = pack_bf16(p2, p3);
                    wpk[e / 2] = MODE == MASK_NONE ? pb[e / 2] : pb[e / 2] & rgo_attn::keep_pair_mask(ksh, e);
                    wpk[e / 2 + 1] =
                        MODE == MASK_NONE ? pb[e / 2 + 1] : pb[e / 2 + 1] & rgo_attn::keep_pair_mask(ksh, e + 2);
                }
                tmem_st16(tS, wpk);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(p_full));
            mbar_wait(smem_u32(dp_full), i & 1);
            tc_fence_after();
            {
                uint32_t d[32];
                tmem_ld32(tdP, d);
                tmem_ld_wait_regs(d);
                uint32_t dpk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    const float4 dd = *reinterpret_cast<const float4*>(Dv + e);
                    const float dv[4] = {dd.x, dd.y, dd.z, dd.w};
                    float ds[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t pw = pb[(e + u) / 2];
                        const float pv = ((e + u) & 1) ? bf16_hi(pw) : bf16_lo(pw);
                        const float dp = ((kw >> (e + u)) & 1u) ? __uint_as_float(d[e + u]) * p.inv_keep : 0.0f;
                        ds[u] = pv * (dp - dv[u]);
                    }
                    dpk[e / 2] = pack_bf16(ds[0], ds[1]);
                    dpk[e / 2 + 1] = pack_bf16(ds[2], ds[3]);
                }
                tmem_st16(tdP, dpk);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t unit = (4 * h + u) ^ sw;
                    *reinterpret_cast<uint4*>(ds_row + unit * 16) =
                        make_uint4(dpk[4 * u], dpk[4 * u + 1], dpk[4 * u + 2], dpk[4 * u + 3]);
                }
            }
            fence_proxy_async_smem();
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(ds_full));
        }
        // ---- epilogue: dV = acc / keep_prob, dK = acc * scale; dims [64h, 64h+64)
        mbar_wait(smem_u32(acc_full), 0);
        tc_fence_after();
        if (p.dkv_tma) {
            // staged as the SW128 tiles of the output tensor maps in the K (dV) and V (dK)
            // buffers -- every MMA has completed -- then one TMA store per tensor and dims
            // half: coalesced 128-byte rows instead of 32 key rows x 16 bytes per warp store
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {
                const uint32_t tacc = tmem + lane_base + 256 + which * HD;
                const float mul = which == 0 ? p.inv_keep : p.scale;
                uint8_t* line = (which == 0 ? sK : sV) + h * SM::KCHUNK + r * 128;
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    uint32_t o[32];
                    tmem_ld32(tacc + h * 64 + 32 * c, o);
                    tmem_ld_wait_regs(o);
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        pk[e] = pack_bf16(__uint_as_float(o[2 * e]) * mul, __uint_as_float(o[2 * e + 1]) * mul);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const uint32_t unit = static_cast<uint32_t>(4 * c + v) ^ static_cast<uint32_t>(r & 7);
                        *reinterpret_cast<uint4*>(line + unit * 16) =
                            make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                    }
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(2 + h, 128);
            if (qw == 0 && lane == 0) {
                tma_store_4d(&tmdV, smem_u32(sK + h * SM::KCHUNK), h * 64, kv0, hh, bb);
                tma_store_4d(&tmdK, smem_u32(sV + h * SM::KCHUNK), h * 64, kv0, hh, bb);
                bulk_group_commit();
                bulk_group_wait_all();  // complete before the CTA exits (see K5's O store)
            }
        } else {
        const int key = kv0 + r;
        __nv_bfloat16* dv_row = static_cast<__nv_bfloat16*>(p.dV) + bb * p.v_sb + hh * p.v_sh +
                                static_cast<long long>(key_valid ? key : 0) * p.v_ss;
        __nv_bfloat16* dk_row = static_cast<__nv_bfloat16*>(p.dK) + bb * p.k_sb + hh * p.k_sh +
                                static_cast<long long>(key_valid ? key : 0) * p.k_ss;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {
            const uint32_t tacc = tmem + lane_base + 256 + which * HD;
            const float mul = which == 0 ? p.inv_keep : p.scale;
            __nv_bfloat16* dst = which == 0 ? dv_row : dk_row;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                const int col = h * 64 + 32 * c;
                uint32_t o[32];
                tmem_ld32(tacc + col, o);
                tmem_ld_wait_regs(o);
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    pk[e] = pack_bf16(__uint_as_float(o[2 * e]) * mul, __uint_as_float(o[2 * e + 1]) * mul);
                if (key_valid) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
                    for (int v = 0; v < 4; ++v) d4[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                }
            }
        }
        }
    } else if (warp >= 12) {  // ------------------------------------------------- dQ drain
        // thread = head dim (TMEM lane 32*qw + lane), 64 query values per tile
        const uint32_t qw = warp & 3;
        const int hd = static_cast<int>(qw * 32 + lane);
        const bool leader = warp == 12 && lane == 0;
        if constexpr (KT_TMEM) {  // K^T -> TMEM columns [192, 256): lane hd, column c = keys (2c, 2c+1)
            mbar_wait(smem_u32(kv_full), 0);
            // K[key][hd] in the SW128 K-major tile: 64-dim chunk hd/64, row = key (128 B),
            // 16-byte unit (hd%64)/8 XOR (key & 7), element hd%8
            const uint8_t* kcol = sK + (hd >> 6) * SM::KCHUNK + (hd & 7) * 2;
            const uint32_t unit = static_cast<uint32_t>((hd & 63) >> 3);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t kt32[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int k0 = 64 * half + 2 * c;
                    const uint32_t lo = *reinterpret_cast<const uint16_t*>(kcol + k0 * 128 + ((unit ^ (k0 & 7)) << 4));
                    const uint32_t hi =
                        *reinterpret_cast<const uint16_t*>(kcol + (k0 + 1) * 128 + ((unit ^ ((k0 + 1) & 7)) << 4));
                    kt32[c] = lo | (hi << 16);
                }
                tmem_st32(tmem + ((qw * 32) << 16) + 192 + 32 * half, kt32);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(kt_full));
        }
        for (int i = 0; i < n_qt; ++i) {
            const int b = i & 1;                        // staging buffer
            const int tb = DQ_BUFS == 2 ? b : 0;        // TMEM accumulator
            mbar_wait(smem_u32(&dq_full[tb]), (i / DQ_BUFS) & 1);
            tc_fence_after();
#if defined(RGO_BWD_DIAG) && (RGO_BWD_DIAG & 2)  // timing diagnostic: no dQ drain/reduction
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&dq_empty[tb]));
            if (true) continue;
#endif
            uint32_t v0[32], v1[32];
            const uint32_t taddr = tmem + ((qw * 32) << 16) + 128 + 64 * tb;
            tmem_ld32(taddr, v0);
            tmem_ld32(taddr + 32, v1);
            tmem_ld_wait();
            reg_fence(v0);
            reg_fence(v1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&dq_empty[tb]));  // TMEM accumulator free
            if (leader) bulk_wait_read1();  // staging b's previous reduce (tile i-2) read out
            named_bar_sync(1, 128);
            float4* stg = reinterpret_cast<float4*>(smem + SM::STG_OFF + b * SM::STG_BYTES);
#pragma unroll
            for (int qg = 0; qg < 8; ++qg)
                stg[qg * 128 + hd] = make_float4(__uint_as_float(v0[4 * qg]), __uint_as_float(v0[4 * qg + 1]),
                                                 __uint_as_float(v0[4 * qg + 2]), __uint_as_float(v0[4 * qg + 3]));
#pragma unroll
            for (int qg = 0; qg < 8; ++qg)
                stg[(8 + qg) * 128 + hd] = make_float4(__uint_as_float(v1[4 * qg]), __uint_as_float(v1[4 * qg + 1]),
                                                       __uint_as_float(v1[4 * qg + 2]), __uint_as_float(v1[4 * qg + 3]));
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (leader) {
                bulk_reduce_add_f32(p.dq_acc + dq2_tile_base(slice, n_qt, qtile(i)), smem_u32(stg), SM::STG_BYTES);
                bulk_commit();
            }
        }
        if (leader) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

template <int MODE, int R>
static cudaError_t launch_main2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                                const CUtensorMap& dO, const CUtensorMap& m, const CUtensorMap& dk,
                                const CUtensorMap& dv, const Params& p, cudaStream_t s) {
    auto kern = bwd_main2_kernel<MODE, R>;
    if (cudaError_t e = rgo::ensure_dyn_smem(reinterpret_cast<const void*>(kern), Smem2::ALLOC); e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>(p.B) * p.H * p.n_kt;
    kern<<<grid, THREADS, Smem2::ALLOC, s>>>(q, k, v, dO, m, dk, dv, p);
    return cudaGetLastError();
}

template <int HD, int MODE, int R, bool DQ = true>
static cudaError_t launch_main(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                               const CUtensorMap& dO, const Params& p, cudaStream_t s) {
    auto kern = bwd_main_kernel<HD, MODE, R, DQ>;
    if (cudaError_t e = rgo::ensure_dyn_smem(reinterpret_cast<const void*>(kern), Smem<HD>::ALLOC); e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>(p.B) * p.H * p.n_kt;
    kern<<<grid, THREADS, Smem<HD>::ALLOC, s>>>(q, k, v, dO, p);
    return cudaGetLastError();
}


// ============================================================================
// K7 split form for head_dim 128 ("v3", launch_attn_bwd3): dK/dV by
// bwd_main_kernel<128, MODE, R, false> (keys on TMEM lanes, 128-query tiles,
// 4 MMAs per tile, no dQ) and dQ by the kernel below -- one CTA per (slice,
// 128-query tile), queries on TMEM lanes, looping over the key tiles:
//   S  = Q K_j^T    (SS, 128 x 128 x 128)        -> TMEM S[j % 2]
//   dP = dO V_j^T   (SS)                         -> TMEM dP
//   P  = 2^(S scale log2e - lse log2e), dS = P o (keep ? dP / p : 0 - D)
//        (the same elementwise terms as bwd_main; dS bf16 over S[j % 2])
//   dQ += dS K_j    (TS: A = dS from TMEM, B = K_j MN-major)  -> TMEM dQ
// dQ accumulates in TMEM over all keys and is written once: no fp32
// accumulator, no cross-CTA reduction (the 64-query kernel moves 8.6 GB of
// bulk reduce-adds at the Llama2-7B shape), and every MMA is 128 x 128 x 128
// (the N = 64 MMAs of the 64-query kernel re-read K/V per 64 queries).  The
// price is recomputing S and dP (7 MMAs per 128 x 128 block instead of 5).
// TMEM: S0 [0,128) S1 [128,256) dP [256,384) dQ [384,512).
// Warps: 0 TMA (Q, dO once; K 3-stage, V 2-stage rings), 1 MMA, 2-3 idle,
// 4-7 / 8-11: the two column halves (keys [0,64) / [64,128) of each tile) of
// every query row, one thread per row.
// ============================================================================
struct Smem3 {
    static constexpr int CHUNK = 128 * 128;      // 128 rows x 128 B
    static constexpr int TILE = 2 * CHUNK;       // 128 rows x 128 bf16
    static constexpr int K_STAGES = 3;
    static constexpr int V_STAGES = 2;
    static constexpr int Q_OFF = 0;
    static constexpr int DO_OFF = TILE;
    static constexpr int K_OFF = 2 * TILE;
    static constexpr int V_OFF = K_OFF + K_STAGES * TILE;
    static constexpr int BAR_OFF = V_OFF + V_STAGES * TILE;
    static constexpr int BYTES = BAR_OFF + 256;
    static constexpr int ALLOC = BYTES + 1023;
};
constexpr int THREADS3 = 384;

// 64 keep bits of one query row: keys [idx0, idx0 + 64) of the global layout
// (n_valid keys valid from idx0), as two LSB-first words.
template <int MODE, int R>
__device__ __forceinline__ void row_word64(const Params& p, uint64_t idx0, int n_valid, uint32_t (&kw)[2]) {
    kw[0] = row_word<MODE, R>(p, idx0, n_valid);
    kw[1] = row_word<MODE, R>(p, idx0 + 32, n_valid - 32);
}

template <int MODE, int R>
__global__ void __launch_bounds__(THREADS3, 1) bwd_dq3_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                               const __grid_constant__ CUtensorMap tmK,
                                                               const __grid_constant__ CUtensorMap tmV,
                                                               const __grid_constant__ CUtensorMap tmdO,
                                                               const Params p, __nv_bfloat16* __restrict__ dQ,
                                                               long long q_sb, long long q_sh, long long q_ss) {
    using SM = Smem3;
    constexpr int HD = 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* sQ = smem + SM::Q_OFF;
    uint8_t* sdO = smem + SM::DO_OFF;
    uint8_t* sK = smem + SM::K_OFF;
    uint8_t* sV = smem + SM::V_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    uint64_t* q_full = bars;                     // Q + dO
    uint64_t* k_full = bars + 1;                 // [3]
    uint64_t* k_empty = k_full + SM::K_STAGES;   // [3]
    uint64_t* v_full = k_empty + SM::K_STAGES;   // [2]
    uint64_t* v_empty = v_full + SM::V_STAGES;   // [2]
    uint64_t* s_full = v_empty + SM::V_STAGES;   // [2]
    uint64_t* s_free = s_full + 2;               // [2] both halves read S(j)
    uint64_t* dp_full = s_free + 2;
    uint64_t* ds_full = dp_full + 1;
    uint64_t* dq_done = ds_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int qt = blockIdx.x % p.n_qt;
    const int bh = blockIdx.x / p.n_qt;
    const int hh = bh % p.H, bb = bh / p.H;
    const uint64_t slice = static_cast<uint64_t>(bb) * p.H + hh;
    const int q0 = qt * BQ;
    const int n_kt = p.n_kt;

    if (warp == 0 && lane == 0) {
        mbar_init(smem_u32(q_full), 1);
        for (int s2 = 0; s2 < SM::K_STAGES; ++s2) {
            mbar_init(smem_u32(&k_full[s2]), 1);
            mbar_init(smem_u32(&k_empty[s2]), 1);
        }
        for (int s2 = 0; s2 < SM::V_STAGES; ++s2) {
            mbar_init(smem_u32(&v_full[s2]), 1);
            mbar_init(smem_u32(&v_empty[s2]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&s_full[b]), 1);
            mbar_init(smem_u32(&s_free[b]), 8);
        }
        mbar_init(smem_u32(dp_full), 1);
        mbar_init(smem_u32(ds_full), 8);
        mbar_init(smem_u32(dq_done), 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmdO);
    }
    if (warp == 1) tmem_alloc<512>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------------------------------ TMA
        if (elect_one()) {
            const uint32_t qb = smem_u32(q_full);
            mbar_arrive_expect_tx(qb, 2 * SM::TILE);
            for (int c = 0; c < 2; ++c) {
                tma_load_4d(smem_u32(sQ + c * SM::CHUNK), &tmQ, qb, c * 64, q0, hh, bb);
                tma_load_4d(smem_u32(sdO + c * SM::CHUNK), &tmdO, qb, c * 64, q0, hh, bb);
            }
        }
        __syncwarp();
        for (int j = 0; j < n_kt; ++j) {
            const int ks = j % SM::K_STAGES, vs = j % SM::V_STAGES;
            mbar_wait(smem_u32(&k_empty[ks]), ((j / SM::K_STAGES) & 1) ^ 1);
            if (elect_one()) {
                const uint32_t kb = smem_u32(&k_full[ks]);
                mbar_arrive_expect_tx(kb, SM::TILE);
                for (int c = 0; c < 2; ++c)
                    tma_load_4d(smem_u32(sK + ks * SM::TILE + c * SM::CHUNK), &tmK, kb, c * 64, j * BKV, hh, bb);
            }
            __syncwarp();
            mbar_wait(smem_u32(&v_empty[vs]), ((j / SM::V_STAGES) & 1) ^ 1);
            if (elect_one()) {
                const uint32_t vb = smem_u32(&v_full[vs]);
                mbar_arrive_expect_tx(vb, SM::TILE);
                for (int c = 0; c < 2; ++c)
                    tma_load_4d(smem_u32(sV + vs * SM::TILE + c * SM::CHUNK), &tmV, vb, c * 64, j * BKV, hh, bb);
            }
            __syncwarp();
        }
    } else if (warp == 1) {  // ----------------------------------------------------- MMA
        constexpr uint32_t IDESC_S = idesc_make(1, 1, BQ, BKV, 0, 0);  // S, dP: K-major A and B
        constexpr uint32_t IDESC_Q = idesc_make(1, 1, BQ, HD, 0, 1);   // dQ: A TMEM, B MN-major
        const uint64_t q_desc = desc_kmajor_sw128(smem_u32(sQ));
        const uint64_t do_desc = desc_kmajor_sw128(smem_u32(sdO));
        const uint64_t k_desc = desc_kmajor_sw128(smem_u32(sK));
        const uint64_t v_desc = desc_kmajor_sw128(smem_u32(sV));
        const uint64_t k_mdesc = desc_sw128(smem_u32(sK), SM::CHUNK, 1024);
        const uint32_t tdP = tmem + 256, tdQ = tmem + 384;
        auto issue_t = [&](uint32_t d, uint64_t a, uint64_t b) {  // 128 x 128 x HD, K-major A and B
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                const uint32_t off = ((kk >> 2) * SM::CHUNK + (kk & 3) * 32) >> 4;
                mma_f16_ss(d, a + off, b + off, IDESC_S, kk > 0);
            }
        };
        auto issue_s = [&](int j) {
            const int ks = j % SM::K_STAGES;
            mbar_wait(smem_u32(&k_full[ks]), (j / SM::K_STAGES) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_t(tmem + (j & 1) * 128, q_desc, k_desc + ((ks * SM::TILE) >> 4));
                tc_commit(smem_u32(&s_full[j & 1]));
            }
            __syncwarp();
        };
        auto issue_dp = [&](int j) {
            const int vs = j % SM::V_STAGES;
            mbar_wait(smem_u32(&v_full[vs]), (j / SM::V_STAGES) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_t(tdP, do_desc, v_desc + ((vs * SM::TILE) >> 4));
                tc_commit(smem_u32(dp_full));
                tc_commit(smem_u32(&v_empty[vs]));
            }
            __syncwarp();
        };
        mbar_wait(smem_u32(q_full), 0);
        issue_s(0);
        issue_dp(0);
        if (n_kt > 1) issue_s(1);
        for (int j = 0; j < n_kt; ++j) {
            mbar_wait(smem_u32(ds_full), j & 1);
            tc_fence_after();
            if (elect_one()) {  // dQ += dS(j) K_j: dS bf16 pairs over S[j % 2], K_j MN-major
                const int ks = j % SM::K_STAGES;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    mma_f16_ts(tdQ, tmem + (j & 1) * 128 + kk * 8,
                               k_mdesc + ((ks * SM::TILE + kk * 2048) >> 4), IDESC_Q, (j > 0 || kk > 0) ? 1u : 0u);
                tc_commit(smem_u32(&k_empty[ks]));
                if (j + 1 == n_kt) tc_commit(smem_u32(dq_done));
            }
            __syncwarp();
            if (j + 1 < n_kt) issue_dp(j + 1);  // overwrites dP after dQ(j) (in issue order)
            if (j + 2 < n_kt) issue_s(j + 2);   // overwrites S[j % 2] after dQ(j) read dS(j)
        }
    } else if (warp >= 4) {  // --------------------------------------------- P / dS, dQ epilogue
        const int h = (warp - 4) >> 2;               // key half of every tile
        const uint32_t qw = warp & 3;
        const int r = static_cast<int>(qw * 32 + lane);  // query row within the tile
        const int i = q0 + r;
        const bool row_valid = i < p.S;
        const uint32_t lane_base = (qw * 32) << 16;
        const float* rw = p.rows + (slice * p.n_qt + qt) * (2 * BQ);
        const float nl = rw[r], Dr = rw[BQ + r];    // -lse*log2e (-inf for padding rows), rowsum(dO o O)
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nl2 = make_float2(nl, nl);
        const uint64_t row_base = (slice * p.S + static_cast<uint64_t>(row_valid ? i : 0)) * p.S;
        uint32_t kw_next[2] = {0u, 0u};
        if (row_valid) row_word64<MODE, R>(p, row_base + 64 * h, p.S - 64 * h, kw_next);
        for (int j = 0; j < n_kt; ++j) {
            const int kc0 = j * BKV + 64 * h;  // first key of this half
            uint32_t kw[2] = {kw_next[0], kw_next[1]};
            if (row_valid && j + 1 < n_kt) row_word64<MODE, R>(p, row_base + kc0 + BKV, p.S - (kc0 + BKV), kw_next);
            const uint32_t tS = tmem + lane_base + (j & 1) * 128;
            mbar_wait(smem_u32(&s_full[j & 1]), (j >> 1) & 1);
            tc_fence_after();
            uint32_t pb[32];  // P as bf16 pairs (the same rounding as bwd_main)
            {
                uint32_t s0[32], s1[32];
                tmem_ld32(tS + 64 * h, s0);
                tmem_ld32(tS + 64 * h + 32, s1);
                tmem_ld_wait();
                reg_fence(s0);
                reg_fence(s1);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&s_free[j & 1]));
                const int valid = p.S - kc0;  // keys >= valid are padding (last tile only)
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    const float2 t0 = __ffma2_rn(make_float2(__uint_as_float(s0[e]), __uint_as_float(s0[e + 1])), sc2, nl2);
                    const float2 t1 = __ffma2_rn(make_float2(__uint_as_float(s1[e]), __uint_as_float(s1[e + 1])), sc2, nl2);
                    float a0 = ex2_approx(t0.x), a1 = ex2_approx(t0.y), b0 = ex2_approx(t1.x), b1 = ex2_approx(t1.y);
                    if (valid < 64) {  // warp-uniform
                        if (e >= valid) a0 = 0.0f;
                        if (e + 1 >= valid) a1 = 0.0f;
                        if (32 + e >= valid) b0 = 0.0f;
                        if (33 + e >= valid) b1 = 0.0f;
                    }
                    pb[e / 2] = pack_bf16(a0, a1);
                    pb[16 + e / 2] = pack_bf16(b0, b1);
                }
            }
            mbar_wait(smem_u32(dp_full), j & 1);
            tc_fence_after();
            uint32_t dsk[32];
            {
                uint32_t d0[32], d1[32];
                tmem_ld32(tmem + lane_base + 256 + 64 * h, d0);
                tmem_ld32(tmem + lane_base + 256 + 64 * h + 32, d1);
                tmem_ld_wait();
                reg_fence(d0);
                reg_fence(d1);
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    float ds[4];
                    const uint32_t dv[4] = {d0[e], d0[e + 1], d1[e], d1[e + 1]};
                    const uint32_t pw[2] = {pb[e / 2], pb[16 + e / 2]};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int col = (u < 2 ? 0 : 32) + e + (u & 1);
                        const float pv = (u & 1) ? bf16_hi(pw[u >> 1]) : bf16_lo(pw[u >> 1]);
                        const float dp = ((kw[col >> 5] >> (col & 31)) & 1u) ? __uint_as_float(dv[u]) * p.inv_keep : 0.0f;
                        ds[u] = pv * (dp - Dr);
                    }
                    dsk[e / 2] = pack_bf16(ds[0], ds[1]);
                    dsk[16 + e / 2] = pack_bf16(ds[2], ds[3]);
                }
            }
            // dS over S[j % 2] columns [32h, 32h+32): both halves must have read S(j) first
            mbar_wait(smem_u32(&s_free[j & 1]), (j >> 1) & 1);
            tmem_st32(tS + 32 * h, dsk);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(ds_full));
        }
        // ---- epilogue: dQ = scale * acc -> bf16, columns [64h, 64h + 64) of row i
        mbar_wait(smem_u32(dq_done), 0);
        tc_fence_after();
        __nv_bfloat16* dst = dQ + bb * q_sb + hh * q_sh + static_cast<long long>(row_valid ? i : 0) * q_ss;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            const int col = 64 * h + 32 * c;
            uint32_t o[32];
            tmem_ld32(tmem + lane_base + 384 + col, o);
            tmem_ld_wait_regs(o);
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                pk[e] = pack_bf16(__uint_as_float(o[2 * e]) * p.scale, __uint_as_float(o[2 * e + 1]) * p.scale);
            if (row_valid) {
                uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
                for (int v = 0; v < 4; ++v) d4[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int MODE, int R>
static cudaError_t launch_dq3(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& dO,
                              const Params& p, __nv_bfloat16* dQ, long long sb, long long sh, long long ss,
                              cudaStream_t s) {
    auto kern = bwd_dq3_kernel<MODE, R>;
    if (cudaError_t e = rgo::ensure_dyn_smem(reinterpret_cast<const void*>(kern), Smem3::ALLOC); e != cudaSuccess)
        return e;
    const unsigned grid = static_cast<unsigned>(p.B) * p.H * p.n_qt;
    kern<<<grid, THREADS3, Smem3::ALLOC, s>>>(q, k, v, dO, p, dQ, sb, sh, ss);
    return cudaGetLastError();
}

}  // namespace rgo_attn_bwd

namespace rgo {

uint64_t attn_bwd_workspace_bytes(int B, int H, int S, int HD) {
    const uint64_t n_qt = (S + rgo_attn_bwd::BQ - 1) / rgo_attn_bwd::BQ;
    const uint64_t rows = static_cast<uint64_t>(B) * H * n_qt * rgo_attn_bwd::BQ;
    return rows * HD * 4 + rows * 2 * 4;
}

static bool tmap4(CUtensorMap* m, const AttnTensor& t, int B, int H, int S, int HD, uint32_t box_rows = 128) {
    const uint64_t dims[4] = {static_cast<uint64_t>(HD), static_cast<uint64_t>(S), static_cast<uint64_t>(H),
                              static_cast<uint64_t>(B)};
    const uint64_t strides[3] = {static_cast<uint64_t>(t.ss) * 2, static_cast<uint64_t>(t.sh) * 2,
                                 static_cast<uint64_t>(t.sb) * 2};
    const uint32_t box[4] = {64, box_rows, 1, 1};
    return make_tmap(m, t.ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Head-dim-128 backward implementation (RGO_BWD_IMPL, read once per process):
//   2 (default) 64-query tiles, dQ^T double-buffered in TMEM, fp32 bulk reduce-adds
//   3           split: dK/dV kernel (128-query tiles, 4 MMAs) + dQ kernel (dQ in TMEM);
//               also selected per call by RGO_ATTN_BWD_DETERMINISTIC
//   1           128-query tiles with dQ into the dP columns (the head-dim-64 kernel)
static int bwd_impl() {
    static const int v = [] {
        const char* e = getenv("RGO_BWD_IMPL");
        if (e && (e[0] == '1' || e[0] == '2' || e[0] == '3')) return e[0] - '0';
        return getenv("RGO_BWD_V1") ? 1 : 2;
    }();
    return v;
}

static void fill_params(rgo_attn_bwd::Params& p, const AttnBwdJob& j, int n_qt, float* rowbuf, float* dq_acc) {
    using namespace rgo_attn_bwd;
    p.B = j.B; p.H = j.H; p.S = j.S;
    p.n_qt = n_qt;
    p.n_kt = (j.S + BKV - 1) / BKV;
    p.scale = j.scale;
    p.scale_log2 = j.scale * 1.4426950408889634f;
    p.inv_keep = 1.0f / (j.mode == rgo_attn::MASK_NONE ? 1.0f : j.keep_prob);
    p.bits = j.bits;
    p.bits_bytes = j.bits_bytes;
    p.bits_aligned = (j.S % 32) == 0 && (reinterpret_cast<uintptr_t>(j.bits) & 3) == 0;
    p.k0 = static_cast<uint32_t>(j.seed);
    p.k1 = static_cast<uint32_t>(j.seed >> 32);
    p.base_offset = j.base_offset;
    p.thr = static_cast<uint32_t>(j.threshold);
    p.rounds = j.rounds;
    p.rows = rowbuf;
    p.dq_acc = dq_acc;
    p.dK = j.dk.ptr; p.k_sb = j.dk.sb; p.k_sh = j.dk.sh; p.k_ss = j.dk.ss;
    p.dV = j.dv.ptr; p.v_sb = j.dv.sb; p.v_sh = j.dv.sh; p.v_ss = j.dv.ss;
}

// head_dim 128: the 64-query-tile kernel (double-buffered dQ^T in TMEM).
static cudaError_t launch_attn_bwd2(const AttnBwdJob& j, cudaStream_t s) {
    using namespace rgo_attn_bwd;
    CUtensorMap tq, tk, tv, tdo;
    if (!tmap4(&tq, j.q, j.B, j.H, j.S, j.HD, BQ2) || !tmap4(&tk, j.k, j.B, j.H, j.S, j.HD) ||
        !tmap4(&tv, j.v, j.B, j.H, j.S, j.HD) || !tmap4(&tdo, j.dout, j.B, j.H, j.S, j.HD, BQ2))
        return cudaErrorInvalidResourceHandle;
    const int n_qt = (j.S + BQ2 - 1) / BQ2;
    const uint64_t rows = static_cast<uint64_t>(j.B) * j.H * n_qt * BQ2;
    float* dq_acc = static_cast<float*>(j.work);
    float* rowbuf = dq_acc + rows * j.HD;
    cudaError_t e;
    {  // row terms + zeroed fp32 dQ accumulator, one pass
        const unsigned threads = 256;
        const unsigned grid = static_cast<unsigned>((rows * 16 + threads - 1) / threads);
        bwd_prep2_kernel<<<grid, threads, 0, s>>>(static_cast<const __nv_bfloat16*>(j.o.ptr), j.o.sb, j.o.sh, j.o.ss,
                                                  static_cast<const __nv_bfloat16*>(j.dout.ptr), j.dout.sb, j.dout.sh,
                                                  j.dout.ss, j.lse, rowbuf, j.B, j.H, j.S, n_qt,
                                                  reinterpret_cast<float4*>(dq_acc), rows * j.HD / 4);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    Params p{};
    fill_params(p, j, n_qt, rowbuf, dq_acc);
    int mode = j.mode;
    if (mode == rgo_attn::MASK_PHILOX && j.threshold >= (uint64_t{1} << 32)) mode = rgo_attn::MASK_NONE;
    // keep-bit tiles by TMA: the mask as a 2-D byte array [B*H*S rows][S/8 bytes],
    // box = 16 bytes (128 keys) x 64 query rows
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    if (mode == rgo_attn::MASK_BITS && j.S % 128 == 0 && (reinterpret_cast<uintptr_t>(j.bits) & 15) == 0) {
        const uint64_t dims[2] = {static_cast<uint64_t>(j.S) / 8, static_cast<uint64_t>(j.B) * j.H * j.S};
        const uint64_t strides[1] = {static_cast<uint64_t>(j.S) / 8};
        const uint32_t box[2] = {16, static_cast<uint32_t>(2 * BQ2)};
        p.mask_tma = make_tmap(&tm, j.bits, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dims, strides, box,
                               CU_TENSOR_MAP_SWIZZLE_NONE) ? 1 : 0;
    }
    // dK/dV by TMA store (16-byte aligned bases and strides)
    CUtensorMap tdk, tdv;
    std::memset(&tdk, 0, sizeof(tdk));
    std::memset(&tdv, 0, sizeof(tdv));
    auto al16 = [](const AttnOut& t) {
        return (reinterpret_cast<uintptr_t>(t.ptr) & 15) == 0 && t.ss % 8 == 0 && t.sh % 8 == 0 && t.sb % 8 == 0;
    };
    p.dkv_tma = RGO_BWD_DKV_TMA && al16(j.dk) && al16(j.dv) &&
                tmap4(&tdk, AttnTensor{j.dk.ptr, j.dk.sb, j.dk.sh, j.dk.ss}, j.B, j.H, j.S, j.HD) &&
                tmap4(&tdv, AttnTensor{j.dv.ptr, j.dv.sb, j.dv.sh, j.dv.ss}, j.B, j.H, j.S, j.HD);
#define RGO_M2(MODEV, RV) launch_main2<MODEV, RV>(tq, tk, tv, tdo, tm, tdk, tdv, p, s)
    if (mode == rgo_attn::MASK_NONE) e = RGO_M2(rgo_attn::MASK_NONE, 0);
    else if (mode == rgo_attn::MASK_BITS) e = RGO_M2(rgo_attn::MASK_BITS, 0);
    else if (j.rounds == 10) e = RGO_M2(rgo_attn::MASK_PHILOX, 10);
    else if (j.rounds == 7) e = RGO_M2(rgo_attn::MASK_PHILOX, 7);
    else e = RGO_M2(rgo_attn::MASK_PHILOX, 0);
#undef RGO_M2
    if (e != cudaSuccess) return e;
    bwd_dq2_kernel<<<static_cast<unsigned>(static_cast<uint64_t>(j.B) * j.H * n_qt), 256, 0, s>>>(
        dq_acc, static_cast<__nv_bfloat16*>(j.dq.ptr), j.dq.sb, j.dq.sh, j.dq.ss, j.B, j.H, j.S, n_qt, j.scale);
    return cudaGetLastError();
}

// head_dim 128, split form: prep (row terms) -> dK/dV kernel -> dQ kernel.
static cudaError_t launch_attn_bwd3(const AttnBwdJob& j, cudaStream_t s) {
    using namespace rgo_attn_bwd;
    CUtensorMap tq, tk, tv, tdo;
    if (!tmap4(&tq, j.q, j.B, j.H, j.S, j.HD) || !tmap4(&tk, j.k, j.B, j.H, j.S, j.HD) ||
        !tmap4(&tv, j.v, j.B, j.H, j.S, j.HD) || !tmap4(&tdo, j.dout, j.B, j.H, j.S, j.HD))
        return cudaErrorInvalidResourceHandle;
    const int n_qt = (j.S + BQ - 1) / BQ;
    const uint64_t rows = static_cast<uint64_t>(j.B) * j.H * n_qt * BQ;
    float* rowbuf = static_cast<float*>(j.work);  // [rows][2] fits the workspace's first rows*HD*4 bytes
    {
        const unsigned threads = 256;
        const unsigned grid = static_cast<unsigned>((rows + threads - 1) / threads);
        bwd_prep_kernel<<<grid, threads, 0, s>>>(static_cast<const __nv_bfloat16*>(j.o.ptr), j.o.sb, j.o.sh, j.o.ss,
                                                 static_cast<const __nv_bfloat16*>(j.dout.ptr), j.dout.sb, j.dout.sh,
                                                 j.dout.ss, j.lse, rowbuf, nullptr, j.B, j.H, j.S, n_qt, j.HD);
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
    }
    Params p{};
    fill_params(p, j, n_qt, rowbuf, nullptr);
    int mode = j.mode;
    if (mode == rgo_attn::MASK_PHILOX && j.threshold >= (uint64_t{1} << 32)) mode = rgo_attn::MASK_NONE;
    auto* dq = static_cast<__nv_bfloat16*>(j.dq.ptr);
    cudaError_t e;
#define RGO_B3(MODEV, RV)                                                                            \
    {                                                                                                \
        e = launch_main<128, MODEV, RV, false>(tq, tk, tv, tdo, p, s);                               \
        if (e == cudaSuccess) e = launch_dq3<MODEV, RV>(tq, tk, tv, tdo, p, dq, j.dq.sb, j.dq.sh, j.dq.ss, s); \
    }
    if (mode == rgo_attn::MASK_NONE) RGO_B3(rgo_attn::MASK_NONE, 0)
    else if (mode == rgo_attn::MASK_BITS) RGO_B3(rgo_attn::MASK_BITS, 0)
    else if (j.rounds == 10) RGO_B3(rgo_attn::MASK_PHILOX, 10)
    else if (j.rounds == 7) RGO_B3(rgo_attn::MASK_PHILOX, 7)
    else RGO_B3(rgo_attn::MASK_PHILOX, 0)
#undef RGO_B3
    return e;
}

cudaError_t launch_attn_bwd(const AttnBwdJob& j, cudaStream_t s) {
    using namespace rgo_attn_bwd;
    if (j.HD == 128 && (j.deterministic || bwd_impl() == 3)) return launch_attn_bwd3(j, s);
    if (j.HD == 128 && bwd_impl() == 2) return launch_attn_bwd2(j, s);
    CUtensorMap tq, tk, tv, tdo;
    if (!tmap4(&tq, j.q, j.B, j.H, j.S, j.HD) || !tmap4(&tk, j.k, j.B, j.H, j.S, j.HD) ||
        !tmap4(&tv, j.v, j.B, j.H, j.S, j.HD) || !tmap4(&tdo, j.dout, j.B, j.H, j.S, j.HD))
        return cudaErrorInvalidResourceHandle;  // tensor-map encode rejected a view
    const int n_qt = (j.S + BQ - 1) / BQ;
    const uint64_t rows = static_cast<uint64_t>(j.B) * j.H * n_qt * BQ;
    float* dq_acc = static_cast<float*>(j.work);
    float* rowbuf = dq_acc + rows * j.HD;
    {
        const unsigned threads = 256;
        const unsigned grid = static_cast<unsigned>((rows + threads - 1) / threads);
        bwd_prep_kernel<<<grid, threads, 0, s>>>(static_cast<const __nv_bfloat16*>(j.o.ptr), j.o.sb, j.o.sh, j.o.ss,
                                                 static_cast<const __nv_bfloat16*>(j.dout.ptr), j.dout.sb, j.dout.sh,
                                                 j.dout.ss, j.lse, rowbuf, dq_acc, j.B, j.H, j.S, n_qt, j.HD);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    Params p{};
    p.B = j.B; p.H = j.H; p.S = j.S;
    p.n_qt = n_qt;
    p.n_kt = (j.S + BKV - 1) / BKV;
    p.scale = j.scale;
    p.scale_log2 = j.scale * 1.4426950408889634f;
    p.inv_keep = 1.0f / (j.mode == rgo_attn::MASK_NONE ? 1.0f : j.keep_prob);
    p.bits = j.bits;
    p.bits_bytes = j.bits_bytes;
    p.bits_aligned = (j.S % 32) == 0 && (reinterpret_cast<uintptr_t>(j.bits) & 3) == 0;
    p.k0 = static_cast<uint32_t>(j.seed);
    p.k1 = static_cast<uint32_t>(j.seed >> 32);
    p.base_offset = j.base_offset;
    p.thr = static_cast<uint32_t>(j.threshold);
    p.rounds = j.rounds;
    p.rows = rowbuf;
    p.dq_acc = dq_acc;
    p.dK = j.dk.ptr; p.k_sb = j.dk.sb; p.k_sh = j.dk.sh; p.k_ss = j.dk.ss;
    p.dV = j.dv.ptr; p.v_sb = j.dv.sb; p.v_sh = j.dv.sh; p.v_ss = j.dv.ss;
    int mode = j.mode;
    if (mode == rgo_attn::MASK_PHILOX && j.threshold >= (uint64_t{1} << 32)) mode = rgo_attn::MASK_NONE;
    cudaError_t e = cudaErrorInvalidValue;
#define RGO_B(HDV, MODEV, RV) \
    if (j.HD == HDV && mode == MODEV) { e = launch_main<HDV, MODEV, RV>(tq, tk, tv, tdo, p, s); goto launched; }
    RGO_B(128, MASK_NONE, 0)
    RGO_B(64, MASK_NONE, 0)
    RGO_B(128, MASK_BITS, 0)
    RGO_B(64, MASK_BITS, 0)
    if (mode == rgo_attn::MASK_PHILOX) {
        if (j.rounds == 10) {
            RGO_B(128, MASK_PHILOX, 10)
            RGO_B(64, MASK_PHILOX, 10)
        } else if (j.rounds == 7) {
            RGO_B(128, MASK_PHILOX, 7)
            RGO_B(64, MASK_PHILOX, 7)
        } else {
            RGO_B(128, MASK_PHILOX, 0)
            RGO_B(64, MASK_PHILOX, 0)
        }
    }
#undef RGO_B
    return cudaErrorNotSupported;
launched:
    if (e != cudaSuccess) return e;
    {
        const unsigned threads = 256;
        const uint64_t n = rows * (j.HD / 8);
        const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
        bwd_dq_kernel<<<grid, threads, 0, s>>>(dq_acc, static_cast<__nv_bfloat16*>(j.dq.ptr), j.dq.sb, j.dq.sh,
                                               j.dq.ss, j.B, j.H, j.S, n_qt, j.HD, j.scale);
    }
    return cudaGetLastError();
}

}  // namespace rgo
