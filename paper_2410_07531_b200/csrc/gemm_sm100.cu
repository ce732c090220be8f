// gemm_sm100.cu -- K2/K3: persistent, warp-specialised tcgen05 GEMM for the
// transformer-block projections whose shapes the reference defines
// (proj/include/rgo/workload.hpp:44-52: QKV, Proj, FFN1, FFN2).
//
//   C[M, N] = epilogue( alpha * A[M, K] . B[N, K]^T )      (both K-major)
//
// * A, B: E4M3 (kind::f8f6f4) or BF16 (kind::f16), fp32 accumulate in TMEM.
// * CTA pairs (cluster of 2, tcgen05 cta_group::2): one 256 x 256 output tile
//   per pair and step; each CTA stages its 128 rows of A and its 128 rows of
//   B (half of the tile's N) per 128-byte K slice, the leader CTA issues
//   tcgen05.mma.cta_group::2 (M = 256) that reads both CTAs' shared memory,
//   and each CTA's TMEM receives its 128 rows x 256 columns.  Per SM this
//   halves the B-operand smem/L2 traffic of a 128 x 256 single-CTA tile.
// * 6-stage TMA -> smem ring per CTA (32 KiB/stage, SWIZZLE_128B); both CTAs'
//   TMA loads complete on the leader's `full` barrier (cp.async.bulk.tensor
//   .cta_group::2); MMA completion is multicast to both CTAs' `empty` /
//   `tfull` barriers (tcgen05.commit.cta_group::2 .multicast::cluster).
// * Warp roles (192 threads per CTA): warp 0 = TMA producer, warp 1 = MMA
//   issuer (leader CTA only; one thread issues), warps 2-5 = epilogue (TMEM
//   -> registers -> scale/activation -> bf16 or e4m3 -> global).  Two
//   256-column TMEM accumulators so the epilogue of tile i overlaps the MMAs
//   of tile i+1; the epilogues of both CTAs release an accumulator on the
//   leader's `tempty` barrier.
// * Persistent grid = #SMs (74 pairs), grouped rasterisation (16 M-blocks of
//   256 rows per group) so concurrently running tiles share A and B in L2.
// * Optional co-resident RNG warps (overlap mechanism B): extra warps that
//   drain the dropout-mask work queue (csrc/rng_queue.cuh) while the tensor
//   core runs, using the registers TMEM frees.
#include "gemm_sm100.cuh"

#include <algorithm>
#include <cstdlib>

namespace rgo_gk {  // instantiated in gemm_inst_*.cu
RGO_GEMM_EXTERN(true, EPI_NONE, OUT_BF16)
RGO_GEMM_EXTERN(true, EPI_NONE, OUT_E4M3)
RGO_GEMM_EXTERN(true, EPI_SWIGLU, OUT_E4M3)
RGO_GEMM_EXTERN(true, EPI_SWIGLU, OUT_BF16)
RGO_GEMM_EXTERN(true, EPI_GELU, OUT_E4M3)
RGO_GEMM_EXTERN(true, EPI_GELU, OUT_BF16)
RGO_GEMM_EXTERN(false, EPI_NONE, OUT_BF16)
RGO_GEMM_EXTERN(false, EPI_SWIGLU, OUT_BF16)
RGO_GEMM_EXTERN(false, EPI_GELU, OUT_BF16)
}  // namespace rgo_gk

namespace rgo {

cudaError_t launch_gemm(const GemmJob& j, cudaStream_t s) {
    using namespace rgo_gk;
    const bool fp8 = j.fp8;
    const size_t esz = fp8 ? 1 : 2;
    if ((j.K * esz) % BKB != 0 || j.M <= 0 || j.N <= 0) return cudaErrorInvalidValue;
    if (j.epi == EPI_SWIGLU && j.N % BN != 0) return cudaErrorInvalidValue;
    const CUtensorMapDataType dt = fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta, tb;
    if (j.rb && (j.rb % BM || j.M % j.rb || j.a_rows <= 0)) return cudaErrorInvalidValue;
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(j.K), static_cast<uint64_t>(j.rb ? j.a_rows : j.M)};
        const uint64_t strides[1] = {static_cast<uint64_t>(j.lda) * esz};
        const uint32_t box[2] = {static_cast<uint32_t>(BKB / esz), BM};
        if (!make_tmap(&ta, j.A, dt, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(j.K), static_cast<uint64_t>(j.N)};
        const uint64_t strides[1] = {static_cast<uint64_t>(j.ldb) * esz};
        const uint32_t box[2] = {static_cast<uint32_t>(BKB / esz), BN / 2};
        if (!make_tmap(&tb, j.B, dt, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    Params p{};
    p.M = j.M;
    p.N = j.N;
    p.K = j.K;
    p.tiles_m = (j.M + TILE_M - 1) / TILE_M;
    p.tiles_n = (j.N + BN - 1) / BN;
    p.C = j.C;
    p.ldc = j.ldc;
    p.n_out = j.epi == EPI_SWIGLU ? j.N / 2 : j.N;
    p.alpha = j.alpha;
    p.out_scale = j.out_scale;
    p.pdl = j.pdl ? 1 : 0;
    // Rasterisation group (M-blocks swept together over all N-blocks): the
    // group's A rows stay in L2 while B streams through once per group, so the
    // DRAM reads are A + B * ceil(tiles_m / group_m).  RGO_GEMM_GROUP_M overrides
    // (measurement A/B); 0 = the default.
    static const int group_env = [] {
        const char* e = getenv("RGO_GEMM_GROUP_M");
        return e ? atoi(e) : 0;
    }();
    // Default: as many M-blocks as fit ~32 MB of A (256 rows x K per block) --
    // the measured optimum (scripts/diag/gemm_group_sweep.py, profiles/r02_gemm_raster.md):
    // at Llama2-7B FFN1 DRAM reads 455 -> 290 MB per launch and 0.929 -> 0.910 ms,
    // QKV 283 -> 226 MB and 0.564 -> 0.555 ms; 64 blocks (64 MB) thrash L2 (1 GB).
    const int auto_group = static_cast<int>(
        std::max<long long>(1, std::min<long long>(64, (32ll << 20) / (static_cast<long long>(TILE_M) * j.K * esz))));
    p.group_m = j.group_m > 0 ? j.group_m : (group_env > 0 ? group_env : auto_group);
    p.rb = j.rb;
    p.rstride = j.rstride;
    p.roff = j.roff;
    if (j.rng) p.rng = *j.rng;
    const int tiles = p.tiles_m * p.tiles_n;
    int grid = j.grid > 0 ? j.grid : num_sms();
    if (grid > 2 * tiles) grid = 2 * tiles;
    grid &= ~1;  // whole CTA pairs
    if (grid < 2) grid = 2;
    const bool rng = j.rng != nullptr;
    const int rw = j.rng_warps ? j.rng_warps : RNG_WARPS_IN_GEMM;
#define RGO_G(F, E, O) \
    if (fp8 == F && j.epi == E && j.out == O) return launch_variant<F, E, O>(ta, tb, p, grid, rng, rw, s);
    RGO_G(true, EPI_NONE, OUT_BF16)
    RGO_G(true, EPI_NONE, OUT_E4M3)
    RGO_G(true, EPI_SWIGLU, OUT_E4M3)
    RGO_G(true, EPI_SWIGLU, OUT_BF16)
    RGO_G(true, EPI_GELU, OUT_E4M3)
    RGO_G(true, EPI_GELU, OUT_BF16)
    RGO_G(false, EPI_NONE, OUT_BF16)
    RGO_G(false, EPI_SWIGLU, OUT_BF16)
    RGO_G(false, EPI_GELU, OUT_BF16)
#undef RGO_G
    return cudaErrorInvalidValue;
}

}  // namespace rgo
