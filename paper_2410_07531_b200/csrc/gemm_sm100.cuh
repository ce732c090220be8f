// gemm_sm100.cuh -- the tcgen05 CTA-pair GEMM kernel template (see
// gemm_sm100.cu for the design notes).  Instantiated per (dtype, epilogue,
// output) in gemm_inst_*.cu so the variants compile in parallel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm.h"
#include "philox.cuh"
#include "rgo_internal.h"
#include "rng_queue.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace rgo_gk {

constexpr int BM = 128;        // rows of A per CTA (the pair's tile has 256)
constexpr int TILE_M = 2 * BM; // output tile rows per CTA pair
constexpr int BN = 256;        // output tile columns (each CTA stages BN/2 rows of B)
constexpr int BKB = 128;       // K bytes per stage (64 bf16 / 128 e4m3)
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BKB;
constexpr int B_BYTES = (BN / 2) * BKB;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int GROUP_M = 16;
constexpr int CORE_THREADS = 192;
constexpr uint32_t TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
    int M, N, K;          // N = rows of B; K in elements
    int tiles_m, tiles_n;
    void* C;
    long long ldc;        // elements
    int n_out;            // output columns (N, or N/2 for SwiGLU)
    float alpha;          // dequant scale (sa * sb)
    float out_scale;      // multiply before the output cast (fp8 quantisation)
    // co-resident RNG (mechanism B)
    rgo::RngQueue rng;
    int pdl;              // launched as a programmatic dependent of the previous kernel
    int rb, rstride, roff;  // row blocks (GemmJob::rb): GEMM row r -> A/C row map_row(r)
    int group_m;            // M-blocks per rasterisation group
};

// GEMM row -> row of A and C: contiguous, or blocks of rb rows every rstride
// rows starting at roff (the query-row chunk of every batch item).
__device__ __forceinline__ int map_row(const Params& p, int r) {
    return p.rb ? (r / p.rb) * p.rstride + p.roff + r % p.rb : r;
}

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int group_m, int& mb, int& nb) {
    const int per_group = group_m * tiles_n;
    const int group = tile / per_group;
    const int first_m = group * group_m;
    const int gsize = min(tiles_m - first_m, group_m);
    const int local = tile - group * per_group;
    mb = first_m + local % gsize;
    nb = local / gsize;
}

// Epilogue activations on the SFU: x * rcp(1 + 2^(-x*log2e)) and tanh.approx
// (IEEE division / tanhf cost ~25 instructions per element).
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.0f + tanh_approx(k0 * (x + k1 * x * x * x)));
}

template <int OUT>
__device__ __forceinline__ void store32(void* C, long long ldc, int row, int col, const float (&v)[32]) {
    if constexpr (OUT == OUT_BF16) {
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            packed[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(C) + row * ldc + col);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
    } else {
        uint32_t packed[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const __nv_fp8x2_storage_t lo =
                __nv_cvt_float2_to_fp8x2(make_float2(v[4 * i], v[4 * i + 1]), __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi =
                __nv_cvt_float2_to_fp8x2(make_float2(v[4 * i + 2], v[4 * i + 3]), __NV_SATFINITE, __NV_E4M3);
            packed[i] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(C) + row * ldc + col);
        dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    }
}

template <bool FP8, int EPI, int OUT, int RNG_WARPS>
__global__ void __launch_bounds__(CORE_THREADS + 32 * RNG_WARPS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
    using namespace sm100;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
    uint8_t* smA = smem;
    uint8_t* smB = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;                  // leader: both CTAs' TMA bytes + 2 producer arrivals
    uint64_t* empty = bars + STAGES;        // each CTA: MMA commit (multicast)
    uint64_t* tfull = bars + 2 * STAGES;    // each CTA: accumulator ready (multicast commit)
    uint64_t* tempty = bars + 2 * STAGES + 2;  // leader: 4 epilogue warps x 2 CTAs
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
    volatile int* gemm_done = reinterpret_cast<volatile int*>(tmem_slot + 1);

    // Warp roles.  Co-resident RNG warps (mechanism B) take the LOWEST warp
    // ids: the SM's warp arbiter favours higher ids, so the TMA / MMA-issue /
    // epilogue warps keep priority over the always-ready RNG warps.
    const uint32_t hw_warp = warp_id(), lane = lane_id();
    const bool is_rng_warp = hw_warp < static_cast<uint32_t>(RNG_WARPS);
    const uint32_t warp = is_rng_warp ? CORE_THREADS / 32 + hw_warp : hw_warp - RNG_WARPS;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 2);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(smem_u32(&tfull[a]), 1);
            mbar_init(smem_u32(&tempty[a]), 8);
        }
        *gemm_done = 0;
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) tmem_alloc2<TMEM_COLS>(smem_u32(tmem_slot));
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers and TMEM exist before any cross-CTA traffic
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // leader-CTA addresses of the pair-wide barriers
    const uint32_t full0_leader = mapa_shared(smem_u32(&full[0]), 0);
    const uint32_t tempty0_leader = mapa_shared(smem_u32(&tempty[0]), 0);

    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int num_tiles = p.tiles_m * p.tiles_n;
    const int kblocks = (p.K * (FP8 ? 1 : 2)) / BKB;
    const int bk_elems = FP8 ? BKB : BKB / 2;
    constexpr uint32_t IDESC = FP8 ? idesc_make(0, 0, TILE_M, BN, 0, 0) : idesc_make(1, 1, TILE_M, BN, 0, 0);

    // The next kernel in the stream may launch its CTAs as SMs free up (its RNG
    // warps start draining at once); every role that touches global memory
    // written or read by the previous kernel waits for it first.
    griddep_launch_dependents();
    if (warp == 0) {  // ---------------- TMA producer (whole warp loops, one lane issues)
        griddep_wait();
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t sa = smem_u32(smA), sb = smem_u32(smB), eb0 = smem_u32(&empty[0]);
        for (int tile = pair; tile < num_tiles; tile += n_pairs) {
            int mb, nb;
            tile_coords(tile, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
            const int row_a = map_row(p, mb * TILE_M + rank * BM), row_b = nb * BN + rank * (BN / 2);
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(eb0 + 8 * stage, phase ^ 1);
                if (elect_one()) {
                    const uint32_t fb = full0_leader + 8 * stage;
                    if (leader) mbar_arrive_expect_tx(fb, 2 * STAGE_BYTES);
                    tma_load_2d_pair(sa + stage * A_BYTES, &tmA, fb, kb * bk_elems, row_a);
                    tma_load_2d_pair(sb + stage * B_BYTES, &tmB, fb, kb * bk_elems, row_b);
                    if (!leader) mbar_arrive_cluster(fb);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer (leader CTA; whole warp loops, one lane issues)
        if (leader) {
            int stage = 0;
            uint32_t phase = 0, acc = 0, acc_phase = 0;
            // descriptors of stage 0; stage s adds s*STAGE/16 to the start-address field
            const uint64_t ad0 = desc_kmajor_sw128(smem_u32(smA)), bd0 = desc_kmajor_sw128(smem_u32(smB));
            const uint32_t fb0 = smem_u32(&full[0]), eb0 = smem_u32(&empty[0]);
            for (int tile = pair; tile < num_tiles; tile += n_pairs) {
                mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(fb0 + 8 * stage, phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t ad = ad0 + static_cast<uint64_t>(stage * (A_BYTES >> 4));
                        const uint64_t bd = bd0 + static_cast<uint64_t>(stage * (B_BYTES >> 4));
#pragma unroll
                        for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K per stage
                            const uint32_t acc_flag = (kb | k) != 0;
                            if constexpr (FP8)
                                mma2_f8_ss(d, ad + 2 * k, bd + 2 * k, IDESC, acc_flag);
                            else
                                mma2_f16_ss(d, ad + 2 * k, bd + 2 * k, IDESC, acc_flag);
                        }
                        tc_commit2_mc(eb0 + 8 * stage);
                        if (kb == kblocks - 1) tc_commit2_mc(smem_u32(&tfull[acc]));
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp < CORE_THREADS / 32) {  // ---------------- epilogue warps 2..5 (both CTAs)
        griddep_wait();
        const uint32_t q = hw_warp & 3;  // TMEM lane quarter = physical warp id % 4
        const int row_in_tile = static_cast<int>(rank) * BM + q * 32 + lane;
        uint32_t acc = 0, acc_phase = 0;
        for (int tile = pair; tile < num_tiles; tile += n_pairs) {
            int mb, nb;
            tile_coords(tile, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
            mbar_wait(smem_u32(&tfull[acc]), acc_phase);
            tc_fence_after();
            const int row_l = mb * TILE_M + row_in_tile;
            const int row = map_row(p, row_l);
            const uint32_t tbase = tmem_base + ((q * 32) << 16) + acc * BN;
            if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {  // gate cols [32c,32c+32), up cols 128 + [32c, ...)
                    uint32_t g[32], u[32];
                    tmem_ld32(tbase + c * 32, g);
                    tmem_ld32(tbase + 128 + c * 32, u);
                    tmem_ld_wait_regs(g);
                    reg_fence(u);
                    float v[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        v[i] = silu(__uint_as_float(g[i]) * p.alpha) * (__uint_as_float(u[i]) * p.alpha) *
                               p.out_scale;
                    const int col = nb * (BN / 2) + c * 32;
                    if (row_l < p.M && col < p.n_out) store32<OUT>(p.C, p.ldc, row, col, v);
                }
            } else {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tbase + c * 32, r);
                    tmem_ld_wait_regs(r);
                    float v[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        float x = __uint_as_float(r[i]) * p.alpha;
                        if constexpr (EPI == EPI_GELU) x = gelu_tanh(x);
                        v[i] = x * p.out_scale;
                    }
                    const int col = nb * BN + c * 32;
                    if (row_l < p.M && col < p.n_out) store32<OUT>(p.C, p.ldc, row, col, v);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty0_leader + 8 * acc);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    } else {
        // ---------------- co-resident RNG warps (mechanism B)
        if constexpr (RNG_WARPS > 0) rgo::rng_queue_drain(p.rng, gemm_done, 4);
    }
    if constexpr (RNG_WARPS > 0) {
        // GEMM roles signal completion so RNG warps stop pulling new chunks.
        if (warp >= 2 && warp < CORE_THREADS / 32) {
            // epilogue warps finish last among GEMM roles
            __syncwarp();
            if (lane == 0) atomicAdd(const_cast<int*>(gemm_done), 1);
        }
    }
    tc_fence_before();
    cluster_sync_all();  // the peer's last MMAs / remote arrivals are done before TMEM goes
    if (warp == 1) tmem_dealloc2<TMEM_COLS>(tmem_base);
}

template <bool FP8, int EPI, int OUT, int RNG_WARPS>
cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid,
                            cudaStream_t s) {
    auto k = gemm_kernel<FP8, EPI, OUT, RNG_WARPS>;
    if (cudaError_t e = rgo::ensure_dyn_smem(reinterpret_cast<const void*>(k), SMEM_BYTES); e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(CORE_THREADS + 32 * RNG_WARPS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k, ta, tb, p);
}

// One (dtype, epilogue, output) variant with its RNG-warp counts.
template <bool F, int E, int O>
cudaError_t launch_variant(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, int grid, bool rng,
                           int rw, cudaStream_t s) {
    if (!rng) return launch_t<F, E, O, 0>(ta, tb, p, grid, s);
    if (rw == 6) return launch_t<F, E, O, 6>(ta, tb, p, grid, s);
    if (rw == 8) return launch_t<F, E, O, 8>(ta, tb, p, grid, s);
    if (rw == 12) return launch_t<F, E, O, 12>(ta, tb, p, grid, s);
    if (rw == 16) return launch_t<F, E, O, 16>(ta, tb, p, grid, s);
    return launch_t<F, E, O, 4>(ta, tb, p, grid, s);
}

#define RGO_GEMM_EXTERN(F, E, O)                                                                                   \
    extern template cudaError_t launch_variant<F, E, O>(const CUtensorMap&, const CUtensorMap&, const Params&, int, \
                                                        bool, int, cudaStream_t);

#define RGO_GEMM_VARIANT(F, E, O)                                                                             \
    template cudaError_t launch_variant<F, E, O>(const CUtensorMap&, const CUtensorMap&, const Params&, int, \
                                                 bool, int, cudaStream_t);

}  // namespace rgo_gk