// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM with 4/8/16 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2410_07531_b200/csrc ldtm_rate.cu -o ldtm_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"
using namespace sm100;

__global__ void k(int iters, int* out) {
    __shared__ uint32_t slot;
    const uint32_t warp = warp_id();
    if (warp == 0) tmem_alloc<512>(smem_u32(&slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + ((it * 32 + (warp >> 2) * 128) & 511), r);
        tmem_ld_wait_regs(r);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= r[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    if (acc == 0x12345 && out) out[0] = acc;
}

int main() {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int warps : {4, 8, 16}) {
        int iters = 20000;
        k<<<148, 32 * warps>>>(10, nullptr);
        cudaEventRecord(a);
        k<<<148, 32 * warps>>>(iters, nullptr);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = 148.0 * warps * iters * 32 * 32 * 4;
        printf("warps=%2d: %.1f TB/s total, %.1f B/ns/SM (%s)\n", warps, bytes / ms / 1e9, bytes / ms / 1e6 / 148,
               cudaGetErrorString(cudaGetLastError()));
    }
}
