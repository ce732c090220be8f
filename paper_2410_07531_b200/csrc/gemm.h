// gemm.h -- internal GEMM / RNG-queue launch interface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "rgo_internal.h"

namespace rgo_gk {
enum { EPI_NONE = 0, EPI_SWIGLU = 1, EPI_GELU = 2 };
enum { OUT_BF16 = 0, OUT_E4M3 = 1 };
constexpr int RNG_WARPS_IN_GEMM = 8;  // default co-resident RNG warps per GEMM CTA (mechanism B)
}  // namespace rgo_gk

namespace rgo {

// Dropout-mask work queue shared by the GEMM-resident RNG warps and the
// tail/stand-alone queue kernel.  Unit = one 16-byte vector (128 elements);
// *counter (device, zeroed before the first producer) hands out chunks of
// 64 vectors (two per lane of the claiming warp).
struct RngQueue {
    uint8_t* out;            // packed mask, 16-byte aligned
    uint64_t n_vec;          // elems / 128 (elems % 128 == 0 required)
    uint64_t base_offset;
    uint32_t k0, k1, thr;    // key, threshold (< 2^32)
    int rounds;
    unsigned long long* counter;
    VecWindow win;           // row window of the layout (chunked pipeline); wv == 0: whole layout
};

struct GemmJob {
    bool fp8;                // e4m3 x e4m3 (else bf16 x bf16), fp32 accumulate
    int M, N, K;             // C[M, N'] = epi(alpha * A[M,K] . B[N,K]^T)
    const void* A;
    long long lda;           // elements
    const void* B;
    long long ldb;
    void* C;
    long long ldc;
    int epi;                 // EPI_*; SwiGLU: B rows interleaved per 256-row tile as
                             // [128 gate rows | 128 up rows], output N/2 columns
    int out;                 // OUT_*
    float alpha;             // dequant scale
    float out_scale;         // pre-cast multiplier (fp8 output quantisation)
    int grid;                // 0 = #SMs (persistent)
    const RngQueue* rng;     // non-null: co-resident RNG warps drain this queue
    int rng_warps;           // 4, 6, 8, 12 or 16 (0 = RNG_WARPS_IN_GEMM; the block picks per workload)
    bool pdl;                // programmatic dependent launch after the previous kernel in the stream
    // Row blocks (SQ-chunk pipelining): when rb > 0, GEMM row r (< M) is row
    // (r / rb) * rstride + roff + r % rb of A and C (rb % 128 == 0), and A's
    // tensor map spans a_rows rows.  rb == 0: rows are contiguous.
    int rb, rstride, roff, a_rows;
    int group_m;             // M-blocks (256 rows) per rasterisation group; 0 = default
};

cudaError_t launch_gemm(const GemmJob& j, cudaStream_t s);
cudaError_t launch_rng_queue(const RngQueue& q, unsigned grid, unsigned block, size_t dyn_smem,
                             cudaStream_t s, bool pdl = false);

}  // namespace rgo
