// block.cu -- transformer-block runtime: the paper's timeline on silicon.
//
// One block = QKV GEMM -> attention -> Proj GEMM -> FFN1 GEMM -> FFN2 GEMM
// (proj/include/rgo/workload.hpp:3-6, :44-52; LayerNorm/residual omitted as
// in the reference); MoE blocks run dispatch -> E x (FFN1, FFN2) -> combine
// in place of the FFN (balanced synthetic routing, BASELINE configs[3]).  A "step" is the steady-state rotation
//     [Proj, FFN1, FFN2 of block L-1, QKV of block L]  ->  attention of block L
// so the four GEMMs between consecutive attention layers form the window the
// RNG hides under (schedule.hpp:111-136):
//   SERIAL_FUSED  baseline: GEMMs, then attention with Philox inline (K6)
//   STREAMS       mechanism A: mask kernel (K1) on a low-priority stream with a
//                 grid capped to co-reside with the GEMM CTAs; GEMMs on a
//                 high-priority stream; attention (K5) waits on an event
//   IN_GEMM       mechanism B: the GEMMs carry co-resident RNG warps draining
//                 the mask queue (K4); a tail drain finishes any remainder
//   NO_RNG        measurement only: GEMMs + mask-reading attention with no RNG
//                 work at all (the denominator of the hidden fraction)
// Each step is captured once into a CUDA graph and replayed.
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>

#include "attn.h"
#include "block.h"
#include "gemm.h"
#include "rgo_internal.h"

namespace rgo_dev {

// bf16 -> e4m3 (saturating) with a scale; 16 elements per thread.
__global__ void quant_e4m3_kernel(const __nv_bfloat16* __restrict__ in, uint8_t* __restrict__ out, uint64_t n,
                                  float scale) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the Proj GEMM may start its RNG warps
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 16;
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; i < n; i += stride) {
        if (i + 16 <= n) {
            const uint4 a = *reinterpret_cast<const uint4*>(in + i);
            const uint4 b = *reinterpret_cast<const uint4*>(in + i + 8);
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[2 * k]));
                const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[2 * k + 1]));
                const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(make_float2(f0.x * scale, f0.y * scale),
                                                                         __NV_SATFINITE, __NV_E4M3);
                const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(make_float2(f1.x * scale, f1.y * scale),
                                                                         __NV_SATFINITE, __NV_E4M3);
                o[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
            }
            *reinterpret_cast<uint4*>(out + i) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
            for (uint64_t t = i; t < n; ++t)
                out[t] = __nv_cvt_float_to_fp8(__bfloat162float(in[t]) * scale, __NV_SATFINITE, __NV_E4M3);
        }
    }
}

// Row-mapped variant for the SQ-chunk pipeline: row r of the window lives at
// (r / rb) * rstride + roff + r % rb of both in and out (d % 16 == 0).
__global__ void quant_e4m3_rows_kernel(const __nv_bfloat16* __restrict__ in, uint8_t* __restrict__ out, int rows,
                                       int d, int rb, int rstride, int roff, float scale) {
    const int vec = d / 16;
    const uint64_t n = static_cast<uint64_t>(rows) * vec;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / vec), c = static_cast<int>(i % vec);
        const uint64_t off = static_cast<uint64_t>((r / rb) * rstride + roff + r % rb) * d + 16 * c;
        const uint4 a = *reinterpret_cast<const uint4*>(in + off);
        const uint4 b = *reinterpret_cast<const uint4*>(in + off + 8);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[2 * k]));
            const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[2 * k + 1]));
            const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(make_float2(f0.x * scale, f0.y * scale),
                                                                     __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(make_float2(f1.x * scale, f1.y * scale),
                                                                     __NV_SATFINITE, __NV_E4M3);
            o[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        *reinterpret_cast<uint4*>(out + off) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// MoE dispatch: row y1[t] -> xd[slot(t, j)] for every token-expert pair
// p = t*k + j (expert p % E, row p / E of its slice).  16 bytes per thread.
__global__ void moe_dispatch_kernel(const uint8_t* __restrict__ y1, uint8_t* __restrict__ xd, int M, int d, int k,
                                    int E) {
    const int vec = d / 16;
    const uint64_t n = static_cast<uint64_t>(M) * k * vec;
    const int me = M * k / E;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(i / vec), c = static_cast<int>(i % vec);
        const int t = p / k, e = p % E, r = p / E;
        const uint4 v = *reinterpret_cast<const uint4*>(y1 + static_cast<uint64_t>(t) * d + 16 * c);
        *reinterpret_cast<uint4*>(xd + (static_cast<uint64_t>(e) * me + r) * d + 16 * c) = v;
    }
}

// MoE combine: x[t] = e4m3(sum_j ye[slot(t, j)] / k).  8 columns per thread.
__global__ void moe_combine_kernel(const __nv_bfloat16* __restrict__ ye, uint8_t* __restrict__ x, int M, int d,
                                   int k, int E) {
    const int vec = d / 8;
    const uint64_t n = static_cast<uint64_t>(M) * vec;
    const int me = M * k / E;
    const float gate = 1.0f / static_cast<float>(k);
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(i / vec), c = static_cast<int>(i % vec);
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = 0; j < k; ++j) {
            const int p = t * k + j, e = p % E, r = p / E;
            const uint4 v = *reinterpret_cast<const uint4*>(ye + (static_cast<uint64_t>(e) * me + r) * d + 8 * c);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                acc[2 * q] += f.x;
                acc[2 * q + 1] += f.y;
            }
        }
        uint32_t o[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                make_float2(acc[4 * q] * gate, acc[4 * q + 1] * gate), __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                make_float2(acc[4 * q + 2] * gate, acc[4 * q + 3] * gate), __NV_SATFINITE, __NV_E4M3);
            o[q] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        *reinterpret_cast<uint2*>(x + static_cast<uint64_t>(t) * d + 8 * c) = make_uint2(o[0], o[1]);
    }
}

// Tensor-parallel all-reduce over peer memory, two-shot (block_step_tp).
struct TpPeers {
    const void* p[rgo::BlockBuffers::MAX_TP];
};

// Reduce-scatter fused with the next GEMM's quantisation: elements [e0, e0+n)
// of [M, d]: out[e] = e4m3(scale * sum_p part_p[e]), summed in fp32 in rank
// order (every rank reduces its own rows, so the order is fixed).  8 elements
// (16 bytes of every peer's bf16 partial) per thread.
__global__ void tp_reduce_quant_kernel(const TpPeers parts, int tp, uint8_t* __restrict__ out, uint64_t e0,
                                       uint64_t n, float scale) {
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x * 8) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int r = 0; r < tp; ++r) {
            const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(parts.p[r]) + e0 + i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                acc[2 * q] += f.x;
                acc[2 * q + 1] += f.y;
            }
        }
        uint32_t o[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                make_float2(acc[4 * q] * scale, acc[4 * q + 1] * scale), __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                make_float2(acc[4 * q + 2] * scale, acc[4 * q + 3] * scale), __NV_SATFINITE, __NV_E4M3);
            o[q] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        *reinterpret_cast<uint2*>(out + e0 + i) = make_uint2(o[0], o[1]);
    }
}

// All-gather of the reduced rows: rank p's block [p*per, (p+1)*per) bytes of
// every other rank's buffer is copied into dst (16-byte vectors).
__global__ void tp_gather_kernel(const TpPeers src, int tp, int rank, uint8_t* __restrict__ dst, uint64_t per) {
    const uint64_t vec = per / 16, n = vec * (tp - 1);
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        int r = static_cast<int>(i / vec);
        r += r >= rank;
        const uint64_t off = static_cast<uint64_t>(r) * per + (i % vec) * 16;
        *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(src.p[r]) + off);
    }
}

}  // namespace rgo_dev

namespace rgo {

static unsigned stream_grid(uint64_t items) {
    return static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, 148 * 16));
}

cudaError_t launch_quant_e4m3(const void* in, void* out, uint64_t n, float scale, cudaStream_t s) {
    const uint64_t threads = (n + 15) / 16;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((threads + 255) / 256, 148 * 16));
    static bool once = (cudaFuncSetAttribute(rgo_dev::quant_e4m3_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared),
                        true);
    (void)once;
    rgo_dev::quant_e4m3_kernel<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in),
                                                    static_cast<uint8_t*>(out), n, scale);
    return cudaGetLastError();
}

cudaError_t launch_quant_e4m3_rows(const void* in, void* out, int rows, int d, int rb, int rstride, int roff,
                                   float scale, cudaStream_t s) {
    if (d % 16 || rb <= 0) return cudaErrorInvalidValue;
    const uint64_t items = static_cast<uint64_t>(rows) * (d / 16);
    rgo_dev::quant_e4m3_rows_kernel<<<stream_grid(items), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(in), static_cast<uint8_t*>(out), rows, d, rb, rstride, roff, scale);
    return cudaGetLastError();
}

struct Block {
    BlockConfig cfg;
    BlockBuffers buf;
    int mode;
    cudaStream_t s_main = nullptr, s_rng = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_rng = nullptr;  // fork/join inside a step
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;    // ordering against the caller's stream
    // phase timing (recorded inside the graph): [0] step start, [1] after the GEMM
    // window, [2] after the end of the step, [3] right before the attention kernel
    cudaEvent_t ev_t[4] = {nullptr, nullptr, nullptr, nullptr};
    // chunked pipeline: per chunk "mask c ready" (s_rng) and "slot of c free" (s_main)
    static constexpr int MAX_CHUNKS = 64;
    cudaEvent_t ev_chunk[MAX_CHUNKS] = {}, ev_slot[MAX_CHUNKS] = {};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches_per_step = 0;
    bool primed = false;  // chunked: window 0's mask (and window 1's for NO_RNG) generated
};

static bool block_pdl() {  // RGO_BLOCK_PDL=0 turns programmatic dependent launch off (A/B)
    static const bool on = [] {
        const char* e = getenv("RGO_BLOCK_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Programmatic dependent launch inside the chunked pipeline's stages (GEMM
// chain, tail drain -> attention).  RGO_CHUNK_PDL=0 turns it off (A/B); 300-step
// stress runs of every mode, graph and eager, at the Llama2-7B shape give the same
// outputs as plain stream order (scripts/diag/chunk_pdl_stress.py).
static bool chunk_pdl() {
    static const bool on = [] {
        const char* e = getenv("RGO_CHUNK_PDL");
        return !(e && e[0] == '0');
    }();
    return on && block_pdl();
}

static int rng_gemms_attach() {
    static const int n = [] {
        const char* e = getenv("RGO_RNG_GEMMS");
        return e ? atoi(e) : 0;
    }();
    return n;
}

static GemmJob gemm(const BlockConfig& c, int M, int N, int K, const void* A, const void* B, void* C, int epi,
                    int out, float alpha, float out_scale) {
    GemmJob j{};
    j.pdl = block_pdl();
    j.fp8 = true;
    j.M = M; j.N = N; j.K = K;
    j.A = A; j.lda = K; j.B = B; j.ldb = K;
    j.C = C;
    j.ldc = epi == rgo_gk::EPI_SWIGLU ? N / 2 : N;
    j.epi = epi; j.out = out;
    j.alpha = alpha; j.out_scale = out_scale;
    j.grid = 0;
    j.rng = nullptr;
    (void)c;
    return j;
}

// Mechanism B's RNG warps per GEMM CTA when the caller leaves the choice to the
// block (rng_block = 0): scaled with the mask's Philox work per GEMM flop.  On the
// power-capped part more RNG warps barely lengthen the GEMM window but shrink the
// tail drain, while with little mask per flop the extra warps only cost GEMM issue
// slots and power (scripts/diag/block_phases.py, realistic data, PDL chain, modes
// interleaved): Llama2-7B (3.2e-4 elements/flop) 8 / 12 / 16 warps: step 4.01 /
// 3.86 / 3.94 ms; MoE (1.6e-4): 4 / 6 / 8 warps 6.87 / 7.03 / 7.05 ms; GPT-3
// (0.4e-4 at Philox-7): 4 / 6 / 8 warps 3.05 / 3.11 / 3.22 ms.
static int auto_rng_warps(const BlockConfig& c) {
    const double M = static_cast<double>(c.batch) * c.seq, d = static_cast<double>(c.heads) * c.head_dim;
    const double rows_ffn = c.experts > 0 ? M * c.top_k : M;
    const double flops = 2.0 * M * d * 4.0 * d + 2.0 * rows_ffn * d * c.ffn * ((c.gated ? 2 : 1) + 1);
    const double work = static_cast<double>(c.batch) * c.heads * c.seq * static_cast<double>(c.seq) * c.rounds / 10.0;
    const double r = work / flops;
    return r <= 1.8e-4 ? 4 : (r <= 2.6e-4 ? 8 : (r <= 3.5e-4 ? 12 : 16));
}

// Phase-timing events: inside a graph capture they must be external event
// record nodes; in eager mode a plain record.
static cudaError_t record_timing(Block& b, int i, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &st);
    if (e != cudaSuccess) return e;
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(b.ev_t[i], s, cudaEventRecordExternal)
                                               : cudaEventRecord(b.ev_t[i], s);
}

// Enqueue one step on b.s_main (+ b.s_rng); returns #kernels launched.
static cudaError_t enqueue_step(Block& b, int* launches) {
    const BlockConfig& c = b.cfg;
    const BlockBuffers& x = b.buf;
    const int M = c.batch * c.seq, d = c.heads * c.head_dim, F = c.ffn;
    const int n1 = c.gated ? 2 * F : F;
    const uint64_t elems = static_cast<uint64_t>(c.batch) * c.heads * c.seq * static_cast<uint64_t>(c.seq);
    cudaStream_t s = b.s_main;
    int n = 0;
    cudaError_t e;
    RngQueue q{};
    q.out = x.mask;
    q.n_vec = elems / 128;
    q.base_offset = c.base_offset;
    q.k0 = static_cast<uint32_t>(c.seed);
    q.k1 = static_cast<uint32_t>(c.seed >> 32);
    q.thr = static_cast<uint32_t>(c.threshold);
    q.rounds = c.rounds;
    q.counter = x.counter;

    if (b.mode == BLOCK_STREAMS) {  // fork: K1 on the low-priority stream
        if ((e = cudaEventRecord(b.ev_fork, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(b.s_rng, b.ev_fork, 0)) != cudaSuccess) return e;
        MaskJob mj{x.mask, elems, c.seed, c.base_offset, c.threshold, c.rounds};
        // Default shape: one 256-thread CTA per SM (two RNG warps per SMSP):
        // it always fits beside a resident GEMM CTA.  Interleaved sweeps
        // (scripts/sweep_overlap.py) over 64-512 threads and 0.5-2 CTAs per
        // SM: with the 2-SM GEMMs this shape finishes the mask inside the GEMM
        // window without slowing the GEMMs more than it gains.
        LaunchShape ls;
        ls.grid = c.rng_grid ? c.rng_grid : static_cast<unsigned>(num_sms());
        ls.block = c.rng_block ? c.rng_block : 256;
        ls.dyn_smem = c.rng_smem;
        if ((e = launch_mask(mj, ls, b.s_rng)) != cudaSuccess) return e;
        ++n;
        if ((e = cudaEventRecord(b.ev_rng, b.s_rng)) != cudaSuccess) return e;
    } else if (b.mode == BLOCK_IN_GEMM) {
        if ((e = cudaMemsetAsync(x.counter, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
    }
    const RngQueue* rq_all = b.mode == BLOCK_IN_GEMM ? &q : nullptr;
    // IN_GEMM: the first `rng_gemms` GEMMs of the step carry RNG warps (0 = all;
    // RGO_RNG_GEMMS overrides): with little mask per GEMM flop the queue empties
    // inside the first GEMMs and later GEMMs need not pay for idle RNG warps
    const int attach = rng_gemms_attach();
    int gemm_idx = 0;
    auto rq_next = [&]() -> const RngQueue* { return (attach == 0 || gemm_idx++ < attach) ? rq_all : nullptr; };
    if ((e = record_timing(b, 0, s)) != cudaSuccess) return e;
    // attention output of the previous block -> e4m3
    if ((e = launch_quant_e4m3(x.attn_in ? x.attn_in : x.attn_o, x.attn_o8, static_cast<uint64_t>(M) * d, c.s_attn,
                               s)) != cudaSuccess)
        return e;
    ++n;
    GemmJob g;
    g = gemm(c, M, d, d, x.attn_o8, x.wo, x.y1, rgo_gk::EPI_NONE, rgo_gk::OUT_E4M3, c.a_proj, c.s_proj);
    g.rng = rq_next();
    // IN_GEMM: RNG warps per GEMM CTA (4, 6, 8, 12 or 16; 0 = auto_rng_warps)
    const int rw = c.rng_block ? static_cast<int>(c.rng_block) : auto_rng_warps(c);
    g.rng_warps = rw;
    if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
    ++n;
    if (c.experts > 0) {  // MoE FFN: dispatch -> per-expert FFN1/FFN2 -> combine
        const int E = c.experts, k = c.top_k, me = M * k / E;
        rgo_dev::moe_dispatch_kernel<<<stream_grid(static_cast<uint64_t>(M) * k * (d / 16)), 256, 0, s>>>(
            static_cast<const uint8_t*>(x.y1), static_cast<uint8_t*>(x.xd), M, d, k, E);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++n;
        for (int ex = 0; ex < E; ++ex) {
            const uint8_t* xd = static_cast<const uint8_t*>(x.xd) + static_cast<uint64_t>(ex) * me * d;
            uint8_t* h = static_cast<uint8_t*>(x.h) + static_cast<uint64_t>(ex) * me * F;
            g = gemm(c, me, n1, d, xd, static_cast<const uint8_t*>(x.w1) + static_cast<uint64_t>(ex) * n1 * d, h,
                     c.gated ? rgo_gk::EPI_SWIGLU : rgo_gk::EPI_GELU, rgo_gk::OUT_E4M3, c.a_ffn1, c.s_ffn1);
            g.rng = rq_next();
            g.rng_warps = rw;
            if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
            ++n;
            g = gemm(c, me, d, F, h, static_cast<const uint8_t*>(x.w2) + static_cast<uint64_t>(ex) * d * F,
                     static_cast<__nv_bfloat16*>(x.ye) + static_cast<uint64_t>(ex) * me * d, rgo_gk::EPI_NONE,
                     rgo_gk::OUT_BF16, c.a_ffn2, c.s_ffn2);
            g.rng = rq_next();
            g.rng_warps = rw;
            if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
            ++n;
        }
        rgo_dev::moe_combine_kernel<<<stream_grid(static_cast<uint64_t>(M) * (d / 8)), 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(x.ye), static_cast<uint8_t*>(x.x), M, d, k, E);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++n;
    } else {
        g = gemm(c, M, n1, d, x.y1, x.w1, x.h, c.gated ? rgo_gk::EPI_SWIGLU : rgo_gk::EPI_GELU, rgo_gk::OUT_E4M3,
                 c.a_ffn1, c.s_ffn1);
        g.rng = rq_next();
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        g = gemm(c, M, d, F, x.h, x.w2, x.x, rgo_gk::EPI_NONE, rgo_gk::OUT_E4M3, c.a_ffn2, c.s_ffn2);
        g.rng = rq_next();
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
    }
    g = gemm(c, M, 3 * d, d, x.x, x.wqkv, x.qkv, rgo_gk::EPI_NONE, rgo_gk::OUT_BF16, c.a_qkv, 1.0f);
    g.rng = rq_next();
    g.rng_warps = rw;
    if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
    ++n;
    if ((e = record_timing(b, 1, s)) != cudaSuccess) return e;
    if (b.mode == BLOCK_IN_GEMM) {  // tail: whatever the GEMM-resident warps left
        if ((e = launch_rng_queue(q, 0, 0, 0, s, block_pdl())) != cudaSuccess) return e;
        ++n;
    } else if (b.mode == BLOCK_STREAMS) {
        if ((e = cudaStreamWaitEvent(s, b.ev_rng, 0)) != cudaSuccess) return e;
    }
    if ((e = record_timing(b, 3, s)) != cudaSuccess) return e;
    // attention on the QKV GEMM output (token-major [M, 3d]) -> attn_o [M, d]
    AttnJob a{};
    a.B = c.batch; a.H = c.heads; a.S = c.seq; a.HD = c.head_dim;
    a.scale = 1.0f / sqrtf(static_cast<float>(c.head_dim));
    const long long ld = 3LL * d;
    const __nv_bfloat16* qkv = static_cast<const __nv_bfloat16*>(x.qkv);
    a.q = {qkv, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
    a.k = {qkv + d, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
    a.v = {qkv + 2 * d, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
    a.o = {x.attn_o, static_cast<long long>(c.seq) * d, c.head_dim, d};
    a.lse = x.lse;
    a.mode = b.mode == BLOCK_SERIAL_FUSED ? rgo_attn::MASK_PHILOX : rgo_attn::MASK_BITS;
    a.keep_prob = c.keep_prob;
    a.bits = x.mask;
    a.bits_bytes = x.mask_bytes;
    a.seed = c.seed;
    a.base_offset = c.base_offset;
    a.threshold = c.threshold;
    a.rounds = c.rounds;
    // programmatic dependent of the tail drain (IN_GEMM) or of the QKV GEMM (the other
    // modes; in STREAMS mode an event join sits in between and the launch is a normal one)
    a.pdl = block_pdl() && b.mode != BLOCK_STREAMS;
    if ((e = launch_attn_fwd(a, s)) != cudaSuccess) return e;
    ++n;
    if ((e = record_timing(b, 2, s)) != cudaSuccess) return e;
    *launches = n;
    return cudaSuccess;
}

// SQ-chunk pipelined step (chunks = C > 1; pipeline_schedule, schedule.hpp:205-239;
// PAPER.md:254-261): the query rows of every sequence are split into C windows
// of Sc = SQ/C rows.  One step is the C-stage rotation
//     for c: attention(c)  ->  quant + Proj + FFN1 + FFN2 + QKV on window c's rows
// Attention(c) reads the step's input QKV (qkv: Q rows of window c, all keys)
// and the window's compact mask [slice][Sc][SQ] from ring slot c % 2; stage c's
// GEMMs (M = B*Sc rows, row blocks of Sc every SQ rows) write window c of qkv_out.
// The mask of window c+1 (window 0 of the next step after the last stage) is
// generated while stage c's GEMMs run -- by K1 on the low-priority stream
// (STREAMS, after attention(c) has released the slot) or by the GEMMs'
// co-resident RNG warps + tail (IN_GEMM) -- so at most two window masks are live
// (2/C of the full mask; capacity.hpp:51-59).  Every keep bit and Philox counter is
// the full layout's, so attention(c) equals rows [c*Sc, (c+1)*Sc) of the
// unchunked attention bitwise, and the row-tiled GEMMs equal the unchunked
// GEMMs' rows bitwise.
static cudaError_t enqueue_step_chunked(Block& b, int* launches) {
    const BlockConfig& c = b.cfg;
    const BlockBuffers& x = b.buf;
    const int C = c.chunks, S = c.seq, Sc = S / C;
    const int M = c.batch * S, Mc = c.batch * Sc, d = c.heads * c.head_dim, F = c.ffn;
    const int n1 = c.gated ? 2 * F : F;
    const uint64_t win_elems = static_cast<uint64_t>(c.batch) * c.heads * Sc * static_cast<uint64_t>(S);
    const uint64_t win_bytes = win_elems / 8;
    cudaStream_t s = b.s_main;
    int n = 0;
    cudaError_t e;
    if ((e = record_timing(b, 0, s)) != cudaSuccess) return e;
    if (b.mode == BLOCK_IN_GEMM &&
        (e = cudaMemsetAsync(x.counter, 0, sizeof(unsigned long long) * C, s)) != cudaSuccess)
        return e;
    auto queue_for = [&](int w) {  // work queue of window w's mask into slot w % 2
        RngQueue q{};
        q.out = x.mask + (w & 1) * win_bytes;
        q.n_vec = win_elems / 128;
        q.base_offset = c.base_offset;
        q.k0 = static_cast<uint32_t>(c.seed);
        q.k1 = static_cast<uint32_t>(c.seed >> 32);
        q.thr = static_cast<uint32_t>(c.threshold);
        q.rounds = c.rounds;
        q.counter = x.counter + w;
        q.win = make_window(static_cast<uint32_t>(Sc), static_cast<uint32_t>(w * Sc), static_cast<uint32_t>(S));
        return q;
    };
    const int rw = c.rng_block ? static_cast<int>(c.rng_block) : auto_rng_warps(c);
    const long long ld = 3LL * d;
    for (int ch = 0; ch < C; ++ch) {
        const int nxt = (ch + 1) % C;  // window whose mask this stage's GEMMs hide
        const int r0 = ch * Sc;
        if (b.mode == BLOCK_STREAMS && ch > 0 && (e = cudaStreamWaitEvent(s, b.ev_chunk[ch], 0)) != cudaSuccess)
            return e;
        AttnJob a{};
        a.B = c.batch; a.H = c.heads; a.S = S; a.HD = c.head_dim;
        a.Sq = Sc;
        a.q_row0 = r0;
        a.bits_rows = Sc;
        a.scale = 1.0f / sqrtf(static_cast<float>(c.head_dim));
        const __nv_bfloat16* qkv = static_cast<const __nv_bfloat16*>(x.qkv);
        a.q = {qkv + static_cast<long long>(r0) * ld, static_cast<long long>(S) * ld, c.head_dim, ld};
        a.k = {qkv + d, static_cast<long long>(S) * ld, c.head_dim, ld};
        a.v = {qkv + 2 * d, static_cast<long long>(S) * ld, c.head_dim, ld};
        a.o = {static_cast<__nv_bfloat16*>(x.attn_o) + static_cast<long long>(r0) * d, static_cast<long long>(S) * d,
               c.head_dim, d};
        a.lse = x.lse;
        a.mode = b.mode == BLOCK_SERIAL_FUSED ? rgo_attn::MASK_PHILOX : rgo_attn::MASK_BITS;
        a.keep_prob = c.keep_prob;
        a.bits = x.mask + (ch & 1) * win_bytes;
        a.bits_bytes = win_bytes;
        a.seed = c.seed;
        a.base_offset = c.base_offset;
        a.threshold = c.threshold;
        a.rounds = c.rounds;
        // programmatic dependent of the previous stage's tail drain / QKV GEMM (not across
        // the STREAMS event join, and not for the step's first kernel)
        a.pdl = chunk_pdl() && ch > 0 && b.mode != BLOCK_STREAMS;
        if ((e = launch_attn_fwd(a, s)) != cudaSuccess) return e;
        ++n;
        if (b.mode == BLOCK_STREAMS) {  // window nxt's mask: after attention(ch) released slot nxt % 2
            if ((e = cudaEventRecord(b.ev_slot[ch], s)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(b.s_rng, b.ev_slot[ch], 0)) != cudaSuccess) return e;
            MaskJob mj{x.mask + (nxt & 1) * win_bytes, win_elems, c.seed, c.base_offset, c.threshold, c.rounds};
            mj.win_rows = static_cast<uint32_t>(Sc);
            mj.row0 = static_cast<uint32_t>(nxt * Sc);
            mj.seq = static_cast<uint32_t>(S);
            LaunchShape ls;
            ls.grid = c.rng_grid ? c.rng_grid : static_cast<unsigned>(num_sms());
            ls.block = c.rng_block ? c.rng_block : 256;
            ls.dyn_smem = c.rng_smem;
            if ((e = launch_mask(mj, ls, b.s_rng)) != cudaSuccess) return e;
            ++n;
            if ((e = cudaEventRecord(b.ev_chunk[nxt], b.s_rng)) != cudaSuccess) return e;
        }
        RngQueue q = queue_for(nxt);
        const RngQueue* rq = b.mode == BLOCK_IN_GEMM ? &q : nullptr;
        // stage ch's GEMMs on window ch's rows: blocks of Sc rows every S rows from row r0
        auto rows = [&](GemmJob& g) {
            g.rb = Sc; g.rstride = S; g.roff = r0; g.a_rows = M;
            g.pdl = chunk_pdl();
            g.rng = rq;
            g.rng_warps = rw;
        };
        if ((e = launch_quant_e4m3_rows(x.attn_o, x.attn_o8, Mc, d, Sc, S, r0, c.s_attn, s)) != cudaSuccess) return e;
        ++n;
        GemmJob g;
        g = gemm(c, Mc, d, d, x.attn_o8, x.wo, x.y1, rgo_gk::EPI_NONE, rgo_gk::OUT_E4M3, c.a_proj, c.s_proj);
        rows(g);
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        g = gemm(c, Mc, n1, d, x.y1, x.w1, x.h, c.gated ? rgo_gk::EPI_SWIGLU : rgo_gk::EPI_GELU, rgo_gk::OUT_E4M3,
                 c.a_ffn1, c.s_ffn1);
        rows(g);
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        g = gemm(c, Mc, d, F, x.h, x.w2, x.x, rgo_gk::EPI_NONE, rgo_gk::OUT_E4M3, c.a_ffn2, c.s_ffn2);
        rows(g);
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        g = gemm(c, Mc, 3 * d, d, x.x, x.wqkv, x.qkv_out, rgo_gk::EPI_NONE, rgo_gk::OUT_BF16, c.a_qkv, 1.0f);
        rows(g);
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        if (b.mode == BLOCK_IN_GEMM) {  // what the stage's RNG warps left of window nxt
            if ((e = launch_rng_queue(q, 0, 0, 0, s, chunk_pdl())) != cudaSuccess) return e;
            ++n;
        }
    }
    // join: window 0's mask for the next step is complete when the step ends
    if (b.mode == BLOCK_STREAMS && (e = cudaStreamWaitEvent(s, b.ev_chunk[0], 0)) != cudaSuccess) return e;
    // phase split is not meaningful across interleaved stages: [GEMM window] = the whole step
    if ((e = record_timing(b, 1, s)) != cudaSuccess) return e;
    if ((e = record_timing(b, 3, s)) != cudaSuccess) return e;
    if ((e = record_timing(b, 2, s)) != cudaSuccess) return e;
    *launches = n;
    return cudaSuccess;
}

// First chunked step: the mask of window 0 (generated by the previous step's last
// stage in steady state) -- and for NO_RNG, which never generates, windows 0 and 1.
static cudaError_t prime_chunked(Block& b, cudaStream_t s) {
    const BlockConfig& c = b.cfg;
    const int C = c.chunks, S = c.seq, Sc = S / C;
    const uint64_t win_elems = static_cast<uint64_t>(c.batch) * c.heads * Sc * static_cast<uint64_t>(S);
    const int wins = b.mode == BLOCK_NO_RNG ? 2 : (b.mode == BLOCK_SERIAL_FUSED ? 0 : 1);
    for (int w = 0; w < wins; ++w) {
        MaskJob mj{b.buf.mask + w * (win_elems / 8), win_elems, c.seed, c.base_offset, c.threshold, c.rounds};
        mj.win_rows = static_cast<uint32_t>(Sc);
        mj.row0 = static_cast<uint32_t>(w * Sc);
        mj.seq = static_cast<uint32_t>(S);
        if (cudaError_t e = launch_mask(mj, LaunchShape{}, s); e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t block_create(const BlockConfig& cfg, const BlockBuffers& buf, int mode, bool use_graph, Block** out) {
    Block* b = new (std::nothrow) Block();
    if (!b) return cudaErrorMemoryAllocation;
    b->cfg = cfg;
    b->buf = buf;
    b->mode = mode;
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = greatest priority (numerically lowest)
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&b->s_main, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&b->s_rng, cudaStreamNonBlocking, lo);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_rng, cudaEventDisableTiming);
    for (int t = 0; t < 4 && e == cudaSuccess; ++t) e = cudaEventCreate(&b->ev_t[t]);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_out, cudaEventDisableTiming);
    if (cfg.chunks > Block::MAX_CHUNKS) e = cudaErrorInvalidValue;
    for (int t = 0; t < cfg.chunks && cfg.chunks > 1 && e == cudaSuccess; ++t) {
        e = cudaEventCreateWithFlags(&b->ev_chunk[t], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_slot[t], cudaEventDisableTiming);
    }
    if (e == cudaSuccess && use_graph && cfg.tp_size <= 1) {  // TP steps are host-synchronised segments
        // (kernel attributes and tensor maps are host-side calls, legal during capture;
        // no step is executed here, so creating a block never touches its buffers)
        e = cudaStreamBeginCapture(b->s_main, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            cudaError_t e2 = b->cfg.chunks > 1 ? enqueue_step_chunked(*b, &b->launches_per_step)
                                               : enqueue_step(*b, &b->launches_per_step);
            e = cudaStreamEndCapture(b->s_main, &b->graph);
            if (e2 != cudaSuccess) e = e2;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&b->exec, b->graph, 0);
    }
    if (e != cudaSuccess) {
        block_destroy(b);
        return e;
    }
    *out = b;
    return cudaSuccess;
}

// Tensor-parallel step, segment `seg` (0..4) on b.s_main (+ b.s_rng), see block.h.
static cudaError_t enqueue_tp_segment(Block& b, int seg, int* launches) {
    const BlockConfig& c = b.cfg;
    const BlockBuffers& x = b.buf;
    const int tp = c.tp_size, r = c.tp_rank;
    const int Hl = c.heads / tp, Fl = c.ffn / tp;
    const int M = c.batch * c.seq, d = c.heads * c.head_dim, dl = Hl * c.head_dim;
    const int n1l = c.gated ? 2 * Fl : Fl;
    const uint64_t sq2 = static_cast<uint64_t>(c.seq) * c.seq;
    const uint64_t elems = static_cast<uint64_t>(c.batch) * Hl * sq2;  // this rank's compact mask
    VecWindow hw;  // heads [r*Hl, (r+1)*Hl) of every batch item of the global layout
    hw.wv = static_cast<uint64_t>(Hl) * sq2 / 128;
    hw.sv = static_cast<uint64_t>(c.heads) * sq2 / 128;
    hw.ov = static_cast<uint64_t>(r) * Hl * sq2 / 128;
    cudaStream_t s = b.s_main;
    int n = 0;
    cudaError_t e;
    RngQueue q{};
    q.out = x.mask;
    q.n_vec = elems / 128;
    q.base_offset = c.base_offset;
    q.k0 = static_cast<uint32_t>(c.seed);
    q.k1 = static_cast<uint32_t>(c.seed >> 32);
    q.thr = static_cast<uint32_t>(c.threshold);
    q.rounds = c.rounds;
    q.counter = x.counter;
    q.win = hw;
    const RngQueue* rq = b.mode == BLOCK_IN_GEMM ? &q : nullptr;
    const int rw = c.rng_block ? static_cast<int>(c.rng_block) : auto_rng_warps(c);
    rgo_dev::TpPeers parts{}, y1s{}, xs{};
    for (int t = 0; t < tp; ++t) {
        parts.p[t] = x.peer_part[t];
        y1s.p[t] = x.peer_y1[t];
        xs.p[t] = x.peer_x[t];
    }
    const uint64_t rows_el = static_cast<uint64_t>(M / tp) * d;  // elements of one rank's row block
    auto reduce = [&](void* out, float scale) -> cudaError_t {
        rgo_dev::tp_reduce_quant_kernel<<<stream_grid(rows_el / 8), 256, 0, s>>>(
            parts, tp, static_cast<uint8_t*>(out), r * rows_el, rows_el, scale);
        ++n;
        return cudaGetLastError();
    };
    auto gather = [&](const rgo_dev::TpPeers& src, void* dst) -> cudaError_t {
        rgo_dev::tp_gather_kernel<<<stream_grid(rows_el / 16 * (tp - 1)), 256, 0, s>>>(
            src, tp, r, static_cast<uint8_t*>(dst), rows_el);
        ++n;
        return cudaGetLastError();
    };
    GemmJob g;
    switch (seg) {
    case 0:  // quant + Proj (row-parallel: K = this rank's dl columns) -> bf16 partial
        if (b.mode == BLOCK_STREAMS) {
            if ((e = cudaEventRecord(b.ev_fork, s)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(b.s_rng, b.ev_fork, 0)) != cudaSuccess) return e;
            MaskJob mj{x.mask, elems, c.seed, c.base_offset, c.threshold, c.rounds};
            mj.vwin = hw;
            LaunchShape ls;
            ls.grid = c.rng_grid ? c.rng_grid : static_cast<unsigned>(num_sms());
            ls.block = c.rng_block ? c.rng_block : 256;
            ls.dyn_smem = c.rng_smem;
            if ((e = launch_mask(mj, ls, b.s_rng)) != cudaSuccess) return e;
            ++n;
            if ((e = cudaEventRecord(b.ev_rng, b.s_rng)) != cudaSuccess) return e;
        } else if (b.mode == BLOCK_IN_GEMM) {
            if ((e = cudaMemsetAsync(x.counter, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
        }
        if ((e = record_timing(b, 0, s)) != cudaSuccess) return e;
        if ((e = launch_quant_e4m3(x.attn_in ? x.attn_in : x.attn_o, x.attn_o8, static_cast<uint64_t>(M) * dl,
                                   c.s_attn, s)) != cudaSuccess)
            return e;
        ++n;
        g = gemm(c, M, d, dl, x.attn_o8, x.wo, x.peer_part[r], rgo_gk::EPI_NONE, rgo_gk::OUT_BF16, c.a_proj, 1.0f);
        g.rng = rq;
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        break;
    case 1:  // reduce-scatter(Proj) + quantise: this rank's rows of y1
        if ((e = reduce(x.y1, c.s_proj)) != cudaSuccess) return e;
        break;
    case 2:  // all-gather y1, FFN1 (column-parallel) + FFN2 (row-parallel) -> bf16 partial
        if ((e = gather(y1s, x.y1)) != cudaSuccess) return e;
        g = gemm(c, M, n1l, d, x.y1, x.w1, x.h, c.gated ? rgo_gk::EPI_SWIGLU : rgo_gk::EPI_GELU, rgo_gk::OUT_E4M3,
                 c.a_ffn1, c.s_ffn1);
        g.rng = rq;
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        g = gemm(c, M, d, Fl, x.h, x.w2, x.peer_part[r], rgo_gk::EPI_NONE, rgo_gk::OUT_BF16, c.a_ffn2, 1.0f);
        g.rng = rq;
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        break;
    case 3:  // reduce-scatter(FFN2) + quantise: this rank's rows of x
        if ((e = reduce(x.x, c.s_ffn2)) != cudaSuccess) return e;
        break;
    case 4: {  // all-gather x, QKV (column-parallel: this rank's heads) -> attention of its heads
        if ((e = gather(xs, x.x)) != cudaSuccess) return e;
        g = gemm(c, M, 3 * dl, d, x.x, x.wqkv, x.qkv, rgo_gk::EPI_NONE, rgo_gk::OUT_BF16, c.a_qkv, 1.0f);
        g.rng = rq;
        g.rng_warps = rw;
        if ((e = launch_gemm(g, s)) != cudaSuccess) return e;
        ++n;
        if ((e = record_timing(b, 1, s)) != cudaSuccess) return e;
        if (b.mode == BLOCK_IN_GEMM) {
            if ((e = launch_rng_queue(q, 0, 0, 0, s, false)) != cudaSuccess) return e;
            ++n;
        } else if (b.mode == BLOCK_STREAMS) {
            if ((e = cudaStreamWaitEvent(s, b.ev_rng, 0)) != cudaSuccess) return e;
        }
        if ((e = record_timing(b, 3, s)) != cudaSuccess) return e;
        AttnJob a{};
        a.B = c.batch; a.H = Hl; a.S = c.seq; a.HD = c.head_dim;
        a.Hg = c.heads; a.h0 = r * Hl;
        a.scale = 1.0f / sqrtf(static_cast<float>(c.head_dim));
        const long long ld = 3LL * dl;
        const __nv_bfloat16* qkv = static_cast<const __nv_bfloat16*>(x.qkv);
        a.q = {qkv, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
        a.k = {qkv + dl, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
        a.v = {qkv + 2 * dl, static_cast<long long>(c.seq) * ld, c.head_dim, ld};
        a.o = {x.attn_o, static_cast<long long>(c.seq) * dl, c.head_dim, dl};
        a.lse = x.lse;
        a.mode = b.mode == BLOCK_SERIAL_FUSED ? rgo_attn::MASK_PHILOX : rgo_attn::MASK_BITS;
        a.keep_prob = c.keep_prob;
        a.bits = x.mask;
        a.bits_bytes = x.mask_bytes;
        a.seed = c.seed;
        a.base_offset = c.base_offset;
        a.threshold = c.threshold;
        a.rounds = c.rounds;
        a.pdl = false;
        if ((e = launch_attn_fwd(a, s)) != cudaSuccess) return e;
        ++n;
        if ((e = record_timing(b, 2, s)) != cudaSuccess) return e;
        break;
    }
    default:
        return cudaErrorInvalidValue;
    }
    *launches += n;
    return cudaSuccess;
}

int block_tp_size(const Block* b) { return b->cfg.tp_size; }

cudaError_t block_step_tp(Block* b, cudaStream_t stream, TpBarrier barrier, void* ctx, int* launches) {
    if (b->cfg.tp_size < 2 || !barrier) return cudaErrorInvalidValue;
    cudaError_t e;
    if ((e = cudaEventRecord(b->ev_in, stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(b->s_main, b->ev_in, 0)) != cudaSuccess) return e;
    int n = 0;
    for (int seg = 0; seg < 5; ++seg) {
        if ((e = enqueue_tp_segment(*b, seg, &n)) != cudaSuccess) return e;
        if (seg < 4) {  // every rank's segment done before any rank reads what it wrote
            if ((e = cudaStreamSynchronize(b->s_main)) != cudaSuccess) return e;
            barrier(ctx);
        }
    }
    if ((e = cudaEventRecord(b->ev_out, b->s_main)) != cudaSuccess) return e;
    if (launches) *launches = n;
    return cudaStreamWaitEvent(stream, b->ev_out, 0);
}

// Run one step ordered after `stream` (and before later work on it).
cudaError_t block_step(Block* b, cudaStream_t stream, int* launches) {
    if (b->cfg.tp_size > 1) return cudaErrorInvalidValue;  // block_step_tp
    cudaError_t e;
    if ((e = cudaEventRecord(b->ev_in, stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(b->s_main, b->ev_in, 0)) != cudaSuccess) return e;
    int n = 0;
    if (b->cfg.chunks > 1 && !b->primed) {
        if ((e = prime_chunked(*b, b->s_main)) != cudaSuccess) return e;
        b->primed = true;
    }
    if (b->exec) {
        e = cudaGraphLaunch(b->exec, b->s_main);
        n = b->launches_per_step;
    } else {
        e = b->cfg.chunks > 1 ? enqueue_step_chunked(*b, &n) : enqueue_step(*b, &n);
    }
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(b->ev_out, b->s_main)) != cudaSuccess) return e;
    if (launches) *launches = n;
    return cudaStreamWaitEvent(stream, b->ev_out, 0);
}

cudaError_t block_last_timings(Block* b, float* ms2) {
    cudaError_t e = cudaEventSynchronize(b->ev_t[2]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms2[0], b->ev_t[0], b->ev_t[1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms2[1], b->ev_t[1], b->ev_t[2]);
    return e;
}

cudaError_t block_last_timings3(Block* b, float* ms3) {
    cudaError_t e = cudaEventSynchronize(b->ev_t[2]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms3[0], b->ev_t[0], b->ev_t[1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms3[1], b->ev_t[1], b->ev_t[3]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms3[2], b->ev_t[3], b->ev_t[2]);
    return e;
}

void block_destroy(Block* b) {
    if (!b) return;
    if (b->exec) cudaGraphExecDestroy(b->exec);
    if (b->graph) cudaGraphDestroy(b->graph);
    if (b->ev_fork) cudaEventDestroy(b->ev_fork);
    if (b->ev_rng) cudaEventDestroy(b->ev_rng);
    for (int t = 0; t < 4; ++t)
        if (b->ev_t[t]) cudaEventDestroy(b->ev_t[t]);
    if (b->ev_in) cudaEventDestroy(b->ev_in);
    if (b->ev_out) cudaEventDestroy(b->ev_out);
    for (int t = 0; t < Block::MAX_CHUNKS; ++t) {
        if (b->ev_chunk[t]) cudaEventDestroy(b->ev_chunk[t]);
        if (b->ev_slot[t]) cudaEventDestroy(b->ev_slot[t]);
    }
    if (b->s_main) cudaStreamDestroy(b->s_main);
    if (b->s_rng) cudaStreamDestroy(b->s_rng);
    delete b;
}

}  // namespace rgo
