// attn_fwd_sm100.cu -- K5/K6: Blackwell flash-attention forward with dropout.
//
// Replaces attn_detail::forward_impl (proj/include/rgo/ref_attention.hpp:56-92)
// for attention_forward / attention_dropout_fused / attention_dropout_decoupled
// (:108-146).  Same semantics as the reference:
//   * softmax denominator over ALL keys, before dropout (:78-82),
//   * kept weights scaled by 1/keep_prob with keep_prob the float value (:85, :125),
//   * keep bit of (slice s, row i, col j) = element (s*SQ + i)*SQ + j of the
//     global mask layout (mask.hpp:35-39, ref_attention.hpp:141-143).
// One kernel template, MaskSource switch:
//   MASK_NONE    plain forward (attention_forward),
//   MASK_BITS    reads 16 B of the precomputed bitmask per row per 128-key tile
//                (the paper's decoupled path, K5),
//   MASK_PHILOX  regenerates the keep bits inline with Philox-R (the
//                conventional fused baseline, K6; bit-identical keep decisions).
//
// Structure (per CTA: one (b, h) slice x 256 query rows = two 128-row Q tiles):
//   warp 0      TMA producer: Q once, K/V 128-key tiles through 2-stage rings
//   warp 1      MMA issuer: S_w = Q_w K^T (SS, bf16 -> fp32 TMEM) and
//               O_w += P_w V (TS: P from TMEM as bf16, V MN-major from smem)
//   warps 2-5   softmax for Q tile 0 (one thread per row), warps 6-9 tile 1:
//               TMEM S -> online softmax (exp2, lazy rescale when the running
//               max grows by > 8) -> dropout -> P (bf16) back into S's columns.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512) fp32 columns; P_w
// overwrites the first 64 columns of S_w (bf16 pairs).  tcgen05.mma executes
// in issue order, so S_w(j+1) is written only after O_w += P_w(j) V(j) read P.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "attn.h"
#include "philox.cuh"
#include "rgo_internal.h"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace rgo_attn {

using namespace sm100;

constexpr int BQ = 128;  // rows per Q tile (one softmax warpgroup)
constexpr int BKV = 128;
constexpr int KV_STAGES = 2;
constexpr int THREADS = 384;        // 3 warpgroups: control, softmax tile 0, softmax tile 1
constexpr int CTRL_REGS = 56;       // setmaxnreg budget of the control warpgroup
constexpr int SOFTMAX_REGS = 224;   // ... and of each softmax warpgroup (4*56 + 8*224 = 65536/32)
constexpr uint32_t TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units

// MASK_BITS with SQ % 128 == 0: the keep-bit tiles (128 query rows x 16 bytes per
// Q tile and KV step, the mask viewed as a 2-D byte array) arrive by TMA in a ring
// of MSK_STAGES, MSK_STAGES - 1 KV steps ahead, instead of per-thread 16-byte
// loads that touch 32 rows per warp instruction (RGO_FWD_MASK_TMA=0: the loads).
#ifndef RGO_FWD_MASK_TMA
#define RGO_FWD_MASK_TMA 1
#endif
#ifndef RGO_FWD_Q_PREFETCH
#define RGO_FWD_Q_PREFETCH 1
#endif
#ifndef RGO_FWD_O_TMA
#define RGO_FWD_O_TMA 1
#endif
#ifndef RGO_FWD_MASK_BOX_ROWS
#define RGO_FWD_MASK_BOX_ROWS 128  // keep-bit rows per TMA box: one Q tile (128) or both (256: -3% at SQ16K)
#endif
constexpr int MASK_BOX_ROWS = RGO_FWD_MASK_BOX_ROWS;
#ifndef RGO_FWD_MSK_STAGES
#define RGO_FWD_MSK_STAGES 4
#endif
constexpr int MSK_STAGES = RGO_FWD_MSK_STAGES;

template <int HD>
struct Smem {
    static constexpr int CHUNK = 128 * 128;            // one 64-dH (128 B) column block of 128 rows
    static constexpr int TILE = (HD / 64) * CHUNK;     // 128 rows x HD
    static constexpr int Q_OFF = 0;
    static constexpr int K_OFF = 2 * TILE;
    static constexpr int V_OFF = K_OFF + KV_STAGES * TILE;
    static constexpr int MSK_OFF = V_OFF + KV_STAGES * TILE;      // keep-bit tiles: [stage][Q tile][128 rows][16 B]
    static constexpr int BAR_OFF = MSK_OFF + MSK_STAGES * 2 * 2048;
    static constexpr int BYTES = BAR_OFF + 256 + 1024;
};

// Keep bits of 128 consecutive elements starting at global index idx0.
template <int MODE, int R>
__device__ __forceinline__ void keep_bits(const AttnParams& p, uint64_t idx0, uint32_t (&kw)[4]) {
    if constexpr (MODE == MASK_BITS) {
        if (p.bits_aligned) {  // SQ % 128 == 0: one 16-byte load per row per tile
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.bits + (idx0 >> 3)));
            kw[0] = v.x; kw[1] = v.y; kw[2] = v.z; kw[3] = v.w;
        } else {  // general: byte loads + funnel shift
            const uint64_t b0 = idx0 >> 3;
            const uint32_t sh = static_cast<uint32_t>(idx0 & 7);
            uint32_t by[17];
#pragma unroll
            for (int t = 0; t < 17; ++t) by[t] = (b0 + t < p.bits_bytes) ? p.bits[b0 + t] : 0u;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const uint64_t lo = static_cast<uint64_t>(by[4 * w]) | (static_cast<uint64_t>(by[4 * w + 1]) << 8) |
                                    (static_cast<uint64_t>(by[4 * w + 2]) << 16) |
                                    (static_cast<uint64_t>(by[4 * w + 3]) << 24) |
                                    (static_cast<uint64_t>(by[4 * w + 4]) << 32);
                kw[w] = static_cast<uint32_t>(lo >> sh);
            }
        }
    } else if constexpr (MODE == MASK_PHILOX) {
        if ((idx0 & 3) == 0) {  // 32 whole Philox blocks: same code as K1
            const uint64_t ctr = p.base_offset + (idx0 >> 2);
            const uint32_t lo = static_cast<uint32_t>(ctr), hi = static_cast<uint32_t>(ctr >> 32);
            if (R > 0 && lo <= 0xFFFFFFFFu - 31u) {
#pragma unroll
                for (int w = 0; w < 4; ++w)
                    kw[w] = rgo_dev::keep32_nowrap<(R > 0 ? R : 1)>(lo + 8 * w, hi, p.k0, p.k1, p.thr, 0u);
            } else {
#pragma unroll 1
                for (int w = 0; w < 4; ++w) {
                    uint32_t acc = 0;
                    for (int b = 0; b < 8; ++b) {
                        const uint64_t c = ctr + 8 * w + b;
                        const uint4 o = rgo_dev::philox_rt(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32),
                                                           0u, 0u, p.k0, p.k1, p.rounds);
                        acc |= (static_cast<uint32_t>(o.x < p.thr) | (static_cast<uint32_t>(o.y < p.thr) << 1) |
                                (static_cast<uint32_t>(o.z < p.thr) << 2) | (static_cast<uint32_t>(o.w < p.thr) << 3))
                               << (4 * b);
                    }
                    kw[w] = acc;
                }
            }
        } else {  // misaligned row start (SQ % 4 != 0): per-element blocks
#pragma unroll 1
            for (int w = 0; w < 4; ++w) {
                uint32_t acc = 0;
                for (int c = 0; c < 32; ++c) {
                    const uint64_t idx = idx0 + 32 * w + c;
                    const uint64_t ctr = p.base_offset + (idx >> 2);
                    const uint4 o = rgo_dev::philox_rt(static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32),
                                                       0u, 0u, p.k0, p.k1, p.rounds);
                    const uint32_t lane = static_cast<uint32_t>(idx & 3);
                    const uint32_t wd = lane == 0 ? o.x : lane == 1 ? o.y : lane == 2 ? o.z : o.w;
                    acc |= static_cast<uint32_t>(wd < p.thr) << c;
                }
                kw[w] = acc;
            }
        }
    } else {
        kw[0] = kw[1] = kw[2] = kw[3] = 0xFFFFFFFFu;
    }
}

// 2^x on the SFU (MUFU.EX2, flush-to-zero): exp2f() adds range fix-ups that
// cost several ALU instructions per element.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA pipes for a pair (FA4-style MUFU offload): x = n + f with
// n = rint(x) from the 1.5*2^23 magic add, 2^f on [-0.5, 0.5] by a degree-3
// polynomial (max rel. error 7.5e-5, far below bf16 P's 2^-9), 2^n added into
// the exponent field.  x is clamped at -125 so masked (-inf) columns give a
// tiny normal instead of garbage (their V rows are zero).
__device__ __forceinline__ float2 ex2_poly2(float x0, float x1) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    constexpr float c0 = 0.9999280571937561f, c1 = 0.6932610273361206f, c2 = 0.24261116981506348f,
                    c3 = 0.05517161637544632f;
    const float2 x = make_float2(fmaxf(x0, -125.0f), fmaxf(x1, -125.0f));
    const float2 t = __fadd2_rn(x, make_float2(kMagic, kMagic));
    const float2 n = __fadd2_rn(t, make_float2(-kMagic, -kMagic));
    const float2 f = __ffma2_rn(n, make_float2(-1.0f, -1.0f), x);
    float2 p = __ffma2_rn(make_float2(c3, c3), f, make_float2(c2, c2));
    p = __ffma2_rn(p, f, make_float2(c1, c1));
    p = __ffma2_rn(p, f, make_float2(c0, c0));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
// Pairs (of the 16 per 32-column chunk) whose 2^x runs on the FMA pipes: one
// in POLY_EVERY (8: 12.5 %; 4 is 0.5 % faster for the mask-bits kernel but slower for
// the ALU-bound inline-Philox one, and K5 and K6 must share it to stay bitwise equal).  MUFU.EX2 (16/clk/SM) and the tensor core need the same
// ~1024 cycles per 128x128 tile, so shifting a share to the idle FMA pipes
// takes the softmax off the critical path.
#ifndef RGO_POLY_EVERY
#define RGO_POLY_EVERY 8
#endif
constexpr int POLY_EVERY = RGO_POLY_EVERY;

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// Mask-bits prefetch distance in KV tiles (MASK_BITS): the row loads are
// 32 rows apart per warp; two tiles ahead measured 2-3 % faster than one at
// B4 H32 SQ4096 and B1 H32 SQ2K/32K (three: no better; profiles/r02_fwd_experiments.md).
#ifndef RGO_FWD_MASK_AHEAD
#define RGO_FWD_MASK_AHEAD 2
#endif
constexpr int MASK_AHEAD = RGO_FWD_MASK_AHEAD;

#ifdef RGO_FWD_TIMING  // diagnostic builds only: per-CTA phase timestamps
__device__ unsigned long long* g_fwd_dbg = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void dbg_mark(int slot) {
    if (g_fwd_dbg) {
        uint32_t sm;
        asm("mov.u32 %0, %%smid;" : "=r"(sm));
        g_fwd_dbg[blockIdx.x * 8 + slot] = gtimer();
        if (slot == 0) g_fwd_dbg[blockIdx.x * 8 + 7] = sm;
    }
}
#define RGO_DBG_MARK(cond, slot) \
    if (cond) dbg_mark(slot)
#else
#define RGO_DBG_MARK(cond, slot)
#endif

template <int HD, int MODE, int R>
__global__ void __launch_bounds__(THREADS, 1) attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                              const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV,
                                                              const __grid_constant__ CUtensorMap tmM,
                                                              const __grid_constant__ CUtensorMap tmO,
                                                              const AttnParams p) {
    using SM = Smem<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
    uint8_t* sQ = smem + SM::Q_OFF;
    uint8_t* sK = smem + SM::K_OFF;
    uint8_t* sV = smem + SM::V_OFF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + KV_STAGES;
    uint64_t* v_full = k_empty + KV_STAGES;
    uint64_t* v_empty = v_full + KV_STAGES;
    uint64_t* s_full = v_empty + KV_STAGES;  // [2]
    uint64_t* p_full = s_full + 2;           // [2]
    uint64_t* o_done = p_full + 2;           // [2]
    uint64_t* p_half = o_done + 2;           // [2] first 64 P columns in TMEM
    uint64_t* m_full = p_half + 2;           // [MSK_STAGES] keep-bit tiles (MASK_BITS, TMA)
    uint64_t* m_empty = m_full + MSK_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(m_empty + MSK_STAGES);
    static_assert((17 + 2 * MSK_STAGES) * 8 + 4 <= 256, "barrier area");

    const uint32_t warp = warp_id(), lane = lane_id();
    RGO_DBG_MARK(threadIdx.x == 0, 0);
    const int pair = blockIdx.x % p.n_pairs;
    const int bh = blockIdx.x / p.n_pairs;
    const int hh = bh % p.H, bb = bh / p.H;
    const int q0 = pair * 2 * BQ;
    const int n_kv = (p.S + BKV - 1) / BKV;

    if (warp == 0 && lane == 0) {
        mbar_init(smem_u32(q_full), 1);
        for (int s = 0; s < KV_STAGES; ++s) {
            mbar_init(smem_u32(&k_full[s]), 1);
            mbar_init(smem_u32(&k_empty[s]), 1);
            mbar_init(smem_u32(&v_full[s]), 1);
            mbar_init(smem_u32(&v_empty[s]), 1);
        }
        for (int w = 0; w < 2; ++w) {
            mbar_init(smem_u32(&s_full[w]), 1);
            mbar_init(smem_u32(&p_full[w]), 4);
            mbar_init(smem_u32(&o_done[w]), 1);
            mbar_init(smem_u32(&p_half[w]), 4);
        }
        for (int t = 0; t < MSK_STAGES; ++t) {
            mbar_init(smem_u32(&m_full[t]), 1);
            mbar_init(smem_u32(&m_empty[t]), 8);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr int NCH = HD / 64;
    griddep_wait();  // launched as a programmatic dependent: the producers of Q/K/V and the mask are done
    RGO_DBG_MARK(threadIdx.x == 0, 1);

    if (warp < 4) {  // ---------------------------------------------- control warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CTRL_REGS));
        if (warp == 0) {  // TMA producer (whole warp loops, one lane issues)
            const uint32_t qb = smem_u32(q_full);
            if (elect_one()) {
                mbar_arrive_expect_tx(qb, 2 * SM::TILE);
                for (int w = 0; w < 2; ++w)
                    for (int c = 0; c < NCH; ++c)
                        tma_load_4d(smem_u32(sQ + w * SM::TILE + c * SM::CHUNK), &tmQ, qb, c * 64, q0 + w * BQ, hh, bb);
            }
            __syncwarp();
            const bool mtma = MODE == MASK_BITS && p.mask_tma;
            // keep bits of (this CTA's 2 x 128 query rows) x (KV tile t) into ring slot t % MSK_STAGES
            const int mrow = static_cast<int>((static_cast<uint64_t>(bb) * p.H + hh) * p.bits_rows) +
                             (p.bits_rows == p.S ? p.q_row0 : 0) + q0;
            auto load_mask = [&](int t) {
                const int ms = t % MSK_STAGES;
                mbar_wait(smem_u32(&m_empty[ms]), ((t / MSK_STAGES) & 1) ^ 1);
                if (elect_one()) {
                    const uint32_t mb = smem_u32(&m_full[ms]);
                    mbar_arrive_expect_tx(mb, 2 * 2048);
                    if constexpr (MASK_BOX_ROWS == 2 * BQ) {  // both Q tiles' 256 rows in one box
                        tma_load_2d(smem_u32(smem + SM::MSK_OFF + ms * 2 * 2048), &tmM, mb, t * 16, mrow);
                    } else {
                        for (int w = 0; w < 2; ++w)
                            tma_load_2d(smem_u32(smem + SM::MSK_OFF + (ms * 2 + w) * 2048), &tmM, mb, t * 16,
                                        mrow + w * BQ);
                    }
                }
                __syncwarp();
            };
            if (mtma)
                for (int t = 0; t < MSK_STAGES - 1 && t < n_kv; ++t) load_mask(t);
            int ks = 0, vs = 0;
            uint32_t kph = 0, vph = 0;
            for (int j = 0; j < n_kv; ++j) {
                mbar_wait(smem_u32(&k_empty[ks]), kph ^ 1);
                if (elect_one()) {
                    const uint32_t kb = smem_u32(&k_full[ks]);
                    mbar_arrive_expect_tx(kb, SM::TILE);
                    for (int c = 0; c < NCH; ++c)
                        tma_load_4d(smem_u32(sK + ks * SM::TILE + c * SM::CHUNK), &tmK, kb, c * 64, j * BKV, hh, bb);
                }
                __syncwarp();
                if (++ks == KV_STAGES) { ks = 0; kph ^= 1; }
                mbar_wait(smem_u32(&v_empty[vs]), vph ^ 1);
                if (elect_one()) {
                    const uint32_t vb = smem_u32(&v_full[vs]);
                    mbar_arrive_expect_tx(vb, SM::TILE);
                    for (int c = 0; c < NCH; ++c)
                        tma_load_4d(smem_u32(sV + vs * SM::TILE + c * SM::CHUNK), &tmV, vb, c * 64, j * BKV, hh, bb);
                }
                __syncwarp();
                if (++vs == KV_STAGES) { vs = 0; vph ^= 1; }
                if (mtma && j + MSK_STAGES - 1 < n_kv) load_mask(j + MSK_STAGES - 1);
            }
            // Warm L2 for the CTA that will most likely take this SM next (CTAs are dispatched
            // in index order, one per SM): its Q tiles are read by no other CTA, so its
            // pipeline fill would otherwise start with an HBM round trip.
            if (RGO_FWD_Q_PREFETCH && elect_one()) {
                const int nb = blockIdx.x + p.resident;
                if (p.resident > 0 && nb < static_cast<int>(gridDim.x)) {
                    const int npair = nb % p.n_pairs, nbh = nb / p.n_pairs;
                    for (int w = 0; w < 2; ++w)
                        for (int c = 0; c < NCH; ++c)
                            tma_prefetch_l2_4d(&tmQ, c * 64, npair * 2 * BQ + w * BQ, nbh % p.H, nbh / p.H);
                }
            }
            __syncwarp();
        } else if (warp == 1) {  // MMA issuer (whole warp loops, one lane issues)
            constexpr uint32_t IDESC_S = idesc_make(1, 1, BQ, BKV, 0, 0);
            constexpr uint32_t IDESC_O = idesc_make(1, 1, BQ, HD, 0, 1);  // V is MN-major
            const uint64_t q_desc = desc_kmajor_sw128(smem_u32(sQ));
            const uint64_t k_desc = desc_kmajor_sw128(smem_u32(sK));
            // V: MN-major SW128, 8-key groups at 1024 B (SBO), 64-dH chunks at CHUNK (LBO)
            const uint64_t v_desc = desc_sw128(smem_u32(sV), SM::CHUNK, 1024);
            auto issue_s = [&](int w, int ks) {
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t off = ((kk >> 2) * SM::CHUNK + (kk & 3) * 32) >> 4;
                    mma_f16_ss(tmem + w * 128, q_desc + ((w * SM::TILE) >> 4) + off,
                               k_desc + ((ks * SM::TILE) >> 4) + off, IDESC_S, kk > 0);
                }
            };
            // O += P.V in two K halves: keys [0,64) as soon as the softmax warps
            // have written the first 64 P columns (p_half), keys [64,128) after p_full
            auto issue_o = [&](int w, int vs, bool acc, int k_lo, int k_hi) {
#pragma unroll
                for (int kk = k_lo; kk < k_hi; ++kk)
                    mma_f16_ts(tmem + 256 + w * 128, tmem + w * 128 + kk * 8,
                               v_desc + ((vs * SM::TILE + kk * 2048) >> 4), IDESC_O, (acc || kk > 0) ? 1u : 0u);
            };
            mbar_wait(smem_u32(q_full), 0);
            int ks = 0, vs = 0;
            uint32_t kph = 0, vph = 0;
            mbar_wait(smem_u32(&k_full[ks]), kph);
            tc_fence_after();
            if (elect_one()) {
                issue_s(0, ks);
                tc_commit(smem_u32(&s_full[0]));
                issue_s(1, ks);
                tc_commit(smem_u32(&s_full[1]));
                tc_commit(smem_u32(&k_empty[ks]));
            }
            __syncwarp();
            if (++ks == KV_STAGES) { ks = 0; kph ^= 1; }
            for (int j = 0; j < n_kv; ++j) {
                const bool has_next = j + 1 < n_kv;
                mbar_wait(smem_u32(&v_full[vs]), vph);
                if (has_next) mbar_wait(smem_u32(&k_full[ks]), kph);
                tc_fence_after();
                for (int w = 0; w < 2; ++w) {
                    mbar_wait(smem_u32(&p_half[w]), j & 1);
                    tc_fence_after();
                    if (elect_one()) issue_o(w, vs, j > 0, 0, BKV / 32);
                    __syncwarp();
                    mbar_wait(smem_u32(&p_full[w]), j & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        issue_o(w, vs, true, BKV / 32, BKV / 16);
                        if (has_next) {
                            issue_s(w, ks);
                            tc_commit(smem_u32(&s_full[w]));
                        }
                        if (w == 1) {
                            tc_commit(smem_u32(&v_empty[vs]));
                            if (has_next) tc_commit(smem_u32(&k_empty[ks]));
                            if (!has_next) {
                                tc_commit(smem_u32(&o_done[0]));
                                tc_commit(smem_u32(&o_done[1]));
                            }
                        }
                    }
                    __syncwarp();
                }
                if (++vs == KV_STAGES) { vs = 0; vph ^= 1; }
                if (has_next && ++ks == KV_STAGES) { ks = 0; kph ^= 1; }
            }
        }
    } else {  // -------------------------------------------------------- softmax
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SOFTMAX_REGS));
        const int w = (warp - 4) >> 2;
        const uint32_t q = warp & 3;
        const int row = q * 32 + lane;
        const int i = q0 + w * BQ + row;  // query index within the slice
        const bool row_valid = i < p.Sq;
        const uint32_t lane_base = (q * 32) << 16;
        const uint32_t tS = tmem + lane_base + w * 128;
        const uint32_t tO = tmem + lane_base + 256 + w * 128;
        const uint64_t slice = static_cast<uint64_t>(bb) * p.H + hh;
        // bits index (MASK_BITS: the buffer's own row layout) and global element
        // index (MASK_PHILOX: the full layout's counters) of key 0 of this row
        const uint64_t ri = static_cast<uint64_t>(row_valid ? i : 0);
        const uint64_t row_base = MODE == MASK_BITS
                                      ? (slice * p.bits_rows + ri + (p.bits_rows == p.S ? p.q_row0 : 0)) * p.S
                                      : ((static_cast<uint64_t>(bb) * p.Hg + p.h0 + hh) * p.S + p.q_row0 + ri) * p.S;
        float m = -INFINITY, l = 0.0f;
        // MASK_BITS: the 16 bytes of tile j+MASK_AHEAD are loaded while tile j is
        // processed (a ring of MASK_AHEAD register quads)
        uint32_t kw_ring[MASK_AHEAD][4];
#pragma unroll
        for (int a = 0; a < MASK_AHEAD; ++a) {
            kw_ring[a][0] = kw_ring[a][1] = kw_ring[a][2] = kw_ring[a][3] = 0u;
            if (MODE == MASK_BITS && !p.mask_tma && row_valid && a < n_kv)
                keep_bits<MODE, R>(p, row_base + a * BKV, kw_ring[a]);
        }
        for (int j = 0; j < n_kv; ++j) {
            const int j0 = j * BKV;
            uint32_t kw[4];
            if (MODE == MASK_BITS && p.mask_tma) {  // this row's 16 bytes of the TMA'd tile
                const int ms = j % MSK_STAGES;
                mbar_wait(smem_u32(&m_full[ms]), (j / MSK_STAGES) & 1);
                const uint4 v = *reinterpret_cast<const uint4*>(smem + SM::MSK_OFF + (ms * 2 + w) * 2048 + row * 16);
                kw[0] = v.x; kw[1] = v.y; kw[2] = v.z; kw[3] = v.w;
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&m_empty[ms]));  // slot free (the words are in registers)
                if (!row_valid) kw[0] = kw[1] = kw[2] = kw[3] = 0;
            } else if constexpr (MODE == MASK_BITS) {
#pragma unroll
                for (int t = 0; t < 4; ++t) kw[t] = kw_ring[0][t];
#pragma unroll
                for (int a = 0; a + 1 < MASK_AHEAD; ++a)
#pragma unroll
                    for (int t = 0; t < 4; ++t) kw_ring[a][t] = kw_ring[a + 1][t];
                if (row_valid && j + MASK_AHEAD < n_kv)
                    keep_bits<MODE, R>(p, row_base + j0 + MASK_AHEAD * BKV, kw_ring[MASK_AHEAD - 1]);
            } else if (row_valid) {
                keep_bits<MODE, R>(p, row_base + j0, kw);
            } else {
                kw[0] = kw[1] = kw[2] = kw[3] = 0;
            }
            mbar_wait(smem_u32(&s_full[w]), j & 1);
            RGO_DBG_MARK(j == 0 && warp == 4 && lane == 0, 2);
            tc_fence_after();
            uint32_t s[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s[c]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 4; ++c) reg_fence(s[c]);
            const int valid = p.S - j0;  // columns >= valid are padding (last tile only)
            if (valid < BKV) {               // warp-uniform: the slow path runs once per row
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (c * 32 + e >= valid) s[c][e] = __float_as_uint(-INFINITY);
            }
            // raw row max (scale > 0 commutes with max): 3-input FMNMX
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; e += 4) {
                    mx0 = fmaxf(mx0, fmaxf(__uint_as_float(s[c][e]), __uint_as_float(s[c][e + 1])));
                    mx1 = fmaxf(mx1, fmaxf(__uint_as_float(s[c][e + 2]), __uint_as_float(s[c][e + 3])));
                }
            const float m_new = fmaxf(m, fmaxf(mx0, mx1) * p.scale_log2);
            const bool need = m_new > m + RESCALE_THRESHOLD;
            if (__any_sync(0xffffffffu, need)) {
                const float alpha = ex2_approx(m - m_new);  // 0 on the first tile
                if (j > 0) {
#pragma unroll 1
                    for (int c = 0; c < HD / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait_regs(o);
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                        tmem_st32(tO + c * 32, o);
                    }
                }
                l *= alpha;
                m = m_new;
            }
            // p = 2^(s*scale - m): one packed FFMA2 + two MUFU.EX2 per pair; the
            // row sum (over ALL keys, before dropout) with packed FADD2.
            const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
            const float2 nm2 = make_float2(-m, -m);
            float2 rs2 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // P columns [64h, 64h+64) -> TMEM cols [32h, 32h+32)
                uint32_t pk[32];
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = 2 * h + cc;
                    uint32_t ksh[8];  // dropout on packed bf16 pairs (keep_pair_mask, attn.h)
#pragma unroll
                    for (int t = 0; t < 8; ++t) ksh[t] = kw[c] << t;
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const float2 t2 = __ffma2_rn(make_float2(__uint_as_float(s[c][e]), __uint_as_float(s[c][e + 1])),
                                                     sc2, nm2);
                        float p0, p1;
                        if (POLY_EVERY > 0 && (e >> 1) % POLY_EVERY == POLY_EVERY - 1) {
                            const float2 pp = ex2_poly2(t2.x, t2.y);
                            p0 = pp.x;
                            p1 = pp.y;
                        } else {
                            p0 = ex2_approx(t2.x);
                            p1 = ex2_approx(t2.y);
                        }
                        rs2 = __fadd2_rn(rs2, make_float2(p0, p1));
                        __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
                        uint32_t pw = *reinterpret_cast<uint32_t*>(&hv);
                        if (MODE != MASK_NONE) pw &= keep_pair_mask(ksh, e);
                        pk[cc * 16 + (e >> 1)] = pw;
                    }
                }
                tmem_st32(tS + 32 * h, pk);
                if (h == 0) {
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(smem_u32(&p_half[w]));
                }
            }
            const float rs = rs2.x + rs2.y;
            l += rs;
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&p_full[w]));
        }
        // ---------------- epilogue: O / (l * keep_prob) -> bf16 rows
        RGO_DBG_MARK(warp == 4 && lane == 0, 3);
        mbar_wait(smem_u32(&o_done[w]), 0);
        RGO_DBG_MARK(warp == 4 && lane == 0, 4);
        tc_fence_after();
        const float inv = 1.0f / (l * p.keep_prob);
        if (p.o_tma) {
            // O -> bf16 rows staged in shared memory as the SW128 tile of the output tensor
            // map (tile w reuses K ring stage w: every MMA has completed), then one TMA store
            // per 64-column block: coalesced 128-byte rows instead of 32 rows x 16 bytes per
            // warp store (the epilogue was ~3 us of a ~56 us CTA at the Llama2-7B shape)
            uint8_t* stg = sK + w * SM::TILE;
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_ld_wait_regs(o);
                uint32_t packed[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(o[2 * e]) * inv,
                                                             __uint_as_float(o[2 * e + 1]) * inv);
                    packed[e] = *reinterpret_cast<uint32_t*>(&h);
                }
                uint8_t* line = stg + (c >> 1) * SM::CHUNK + row * 128;
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint32_t unit = static_cast<uint32_t>((c & 1) * 4 + v) ^ static_cast<uint32_t>(row & 7);
                    *reinterpret_cast<uint4*>(line + unit * 16) =
                        make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + w, 128);
            if (warp == 4 + 4 * w && lane == 0) {
                for (int cb = 0; cb < HD / 64; ++cb)
                    tma_store_4d(&tmO, smem_u32(stg + cb * SM::CHUNK), cb * 64, q0 + w * BQ, hh, bb);
                bulk_group_commit();
                // the store complete (not only its read of the staging smem) before the CTA
                // exits: with only the read waited for, back-to-back eager block steps with
                // programmatic dependent launch hung (scripts/diag/pdl_stress.py, streams mode)
                bulk_group_wait_all();
            }
        } else {
            __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.O) + bb * p.o_sb + hh * p.o_sh +
                                  static_cast<long long>(row_valid ? i : 0) * p.o_ss;
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_ld_wait_regs(o);
                uint32_t packed[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(o[2 * e]) * inv,
                                                             __uint_as_float(o[2 * e + 1]) * inv);
                    packed[e] = *reinterpret_cast<uint32_t*>(&h);
                }
                if (row_valid) {
                    uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
                }
            }
        }
        if (p.lse && row_valid) p.lse[slice * p.S + p.q_row0 + i] = (m + __log2f(l)) * 0.6931471805599453f;
        RGO_DBG_MARK(warp == 4 && lane == 0, 5);
    }
    __syncthreads();
    RGO_DBG_MARK(threadIdx.x == 0, 6);
    if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

template <int HD, int MODE, int R>
static cudaError_t launch_t(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& m,
                            const CUtensorMap& o, const AttnParams& p, cudaStream_t s, bool pdl) {
    auto kern = attn_fwd_kernel<HD, MODE, R>;
    if (cudaError_t e = rgo::ensure_dyn_smem(reinterpret_cast<const void*>(kern), Smem<HD>::BYTES); e != cudaSuccess)
        return e;
    const unsigned grid = static_cast<unsigned>(p.B) * p.H * p.n_pairs;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Smem<HD>::BYTES;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, q, k, v, m, o, p);
}

}  // namespace rgo_attn

#ifdef RGO_FWD_TIMING
extern "C" int rgo_debug_fwd_timing(unsigned long long* d_buf) {  // diagnostic builds only
    return cudaMemcpyToSymbol(rgo_attn::g_fwd_dbg, &d_buf, sizeof(d_buf)) == cudaSuccess ? 0 : 2;
}
#endif

namespace rgo {

static bool tmap_qkv(CUtensorMap* m, const AttnTensor& t, int B, int H, int S, int HD) {
    const uint64_t dims[4] = {static_cast<uint64_t>(HD), static_cast<uint64_t>(S), static_cast<uint64_t>(H),
                              static_cast<uint64_t>(B)};
    const uint64_t strides[3] = {static_cast<uint64_t>(t.ss) * 2, static_cast<uint64_t>(t.sh) * 2,
                                 static_cast<uint64_t>(t.sb) * 2};
    const uint32_t box[4] = {64, 128, 1, 1};
    return make_tmap(m, t.ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

cudaError_t launch_attn_fwd(const AttnJob& j, cudaStream_t s) {
    using namespace rgo_attn;
    CUtensorMap tq, tk, tv;
    const int Sq = j.Sq > 0 ? j.Sq : j.S;
    if (j.q_row0 < 0 || j.q_row0 + Sq > j.S) return cudaErrorInvalidValue;
    if (!tmap_qkv(&tq, j.q, j.B, j.H, Sq, j.HD) || !tmap_qkv(&tk, j.k, j.B, j.H, j.S, j.HD) ||
        !tmap_qkv(&tv, j.v, j.B, j.H, j.S, j.HD))
        return cudaErrorInvalidValue;
    AttnParams p{};
    p.B = j.B; p.H = j.H; p.S = j.S;
    p.Sq = Sq;
    p.q_row0 = j.q_row0;
    p.bits_rows = j.bits_rows > 0 ? j.bits_rows : j.S;
    if (p.bits_rows != j.S && p.bits_rows != Sq) return cudaErrorInvalidValue;
    p.n_pairs = (Sq + 2 * BQ - 1) / (2 * BQ);
    p.resident = rgo::num_sms();  // one CTA per SM (shared memory, 512 TMEM columns)
    p.scale_log2 = j.scale * 1.4426950408889634f;
    p.keep_prob = j.mode == MASK_NONE ? 1.0f : j.keep_prob;
    p.bits = j.bits;
    p.bits_bytes = j.bits_bytes;
    p.bits_aligned = (j.S % 128) == 0 && (reinterpret_cast<uintptr_t>(j.bits) & 15) == 0;
    p.k0 = static_cast<uint32_t>(j.seed);
    p.k1 = static_cast<uint32_t>(j.seed >> 32);
    p.base_offset = j.base_offset;
    p.thr = static_cast<uint32_t>(j.threshold);
    p.rounds = j.rounds;
    p.O = j.o.ptr;
    p.o_sb = j.o.sb; p.o_sh = j.o.sh; p.o_ss = j.o.ss;
    p.lse = j.lse;
    p.Hg = j.Hg > 0 ? j.Hg : j.H;
    p.h0 = j.Hg > 0 ? j.h0 : 0;
    if (p.h0 < 0 || p.h0 + j.H > p.Hg) return cudaErrorInvalidValue;
    int mode = j.mode;
    // keep-all (threshold 2^32) or keep_prob 1: every bit is 1 -> plain path, scale 1/p
    if (mode == MASK_PHILOX && j.threshold >= (uint64_t{1} << 32)) mode = MASK_NONE;
    // keep-bit tiles by TMA: the mask as a 2-D byte array [B*H*bits_rows rows][S/8 bytes],
    // box = 16 bytes (128 keys) x 128 query rows
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    p.mask_tma = 0;
    if (RGO_FWD_MASK_TMA && mode == MASK_BITS && p.bits_aligned) {
        const uint64_t dims[2] = {static_cast<uint64_t>(j.S) / 8, static_cast<uint64_t>(j.B) * j.H * p.bits_rows};
        const uint64_t strides[1] = {static_cast<uint64_t>(j.S) / 8};
        const uint32_t box[2] = {16, static_cast<uint32_t>(MASK_BOX_ROWS)};
        p.mask_tma = make_tmap(&tm, j.bits, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dims, strides, box,
                               CU_TENSOR_MAP_SWIZZLE_NONE) ? 1 : 0;
    }
    // O by TMA store (16-byte aligned base and strides: the tensor map's requirement)
    CUtensorMap to;
    std::memset(&to, 0, sizeof(to));
    p.o_tma = 0;
    if (RGO_FWD_O_TMA && (reinterpret_cast<uintptr_t>(j.o.ptr) & 15) == 0 && j.o.ss % 8 == 0 && j.o.sh % 8 == 0 &&
        j.o.sb % 8 == 0) {
        const AttnTensor ov{j.o.ptr, j.o.sb, j.o.sh, j.o.ss};
        p.o_tma = tmap_qkv(&to, ov, j.B, j.H, Sq, j.HD) ? 1 : 0;
    }
#define RGO_A(HDV, MODEV, RV) \
    if (j.HD == HDV && mode == MODEV) return launch_t<HDV, MODEV, RV>(tq, tk, tv, tm, to, p, s, j.pdl);
    RGO_A(128, MASK_NONE, 0)
    RGO_A(64, MASK_NONE, 0)
    RGO_A(128, MASK_BITS, 0)
    RGO_A(64, MASK_BITS, 0)
    if (mode == MASK_PHILOX) {
        if (j.rounds == 10) {
            RGO_A(128, MASK_PHILOX, 10)
            RGO_A(64, MASK_PHILOX, 10)
        } else if (j.rounds == 7) {
            RGO_A(128, MASK_PHILOX, 7)
            RGO_A(64, MASK_PHILOX, 7)
        } else if (j.rounds == 5) {  // reduced-round baselines
            RGO_A(128, MASK_PHILOX, 5)
            RGO_A(64, MASK_PHILOX, 5)
        } else if (j.rounds == 3) {
            RGO_A(128, MASK_PHILOX, 3)
            RGO_A(64, MASK_PHILOX, 3)
        } else {
            RGO_A(128, MASK_PHILOX, 0)
            RGO_A(64, MASK_PHILOX, 0)
        }
    }
#undef RGO_A
    return cudaErrorInvalidValue;
}

}  // namespace rgo
