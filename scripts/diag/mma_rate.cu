// Microbenchmark: tcgen05.mma kind::f16 throughput per SM for SS vs TS
// operands and N in {64, 128, 256} (M = 128, cta_group::1), no TMA traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2410_07531_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"
using namespace sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(int iters, int* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const uint32_t warp = warp_id();
    if (warp == 0) tmem_alloc<512>(smem_u32(&slot));
    if (threadIdx.x == 32) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 1) {
        constexpr uint32_t IDESC = idesc_make(1, 1, 128, N, 0, 0);
        const uint64_t a = desc_kmajor_sw128(smem_u32(sm));
        const uint64_t b = desc_kmajor_sw128(smem_u32(sm + 65536));
        if (elect_one()) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (TS) mma_f16_ts(tmem + 256, tmem + 0 + kk * 8, b + ((kk & 3) * 32 >> 4), IDESC, 1);
                    else mma_f16_ss(tmem + 256, a + ((kk & 3) * 32 >> 4), b + ((kk & 3) * 32 >> 4), IDESC, 1);
                }
            }
            tc_commit(smem_u32(&bar));
        }
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    if (threadIdx.x == 0 && iters < 0) out[0] = 1;
}

template <int N, bool TS>
void run() {
    auto kern = k<N, TS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    int iters = 4000;
    kern<<<148, 128, 140000>>>(10, nullptr);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<148, 128, 140000>>>(iters, nullptr);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 148.0 * iters * 8 * 2.0 * 128 * N * 16;
    printf("%s N=%3d: %.1f TFLOP/s  (%s)\n", TS ? "TS" : "SS", N, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<64, false>(); run<128, false>(); run<256, false>();
    run<64, true>(); run<128, true>(); run<256, true>();
}
