// Microbenchmark: Philox round throughput with IMAD.WIDE (ptxas default) vs
// split IMAD.HI + IMAD (operand made opaque so ptxas cannot re-fuse them).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mulwide.cu -o mulwide
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t opaque(uint32_t x) { asm volatile("mov.b32 %0, %0;" : "+r"(x)); return x; }

template <int SPLIT>
__global__ void k(uint32_t* out, uint32_t k0, uint32_t k1, int iters, uint32_t m0o, uint32_t m1o) {
    uint32_t c0 = threadIdx.x, c1 = blockIdx.x, c2 = 7, c3 = 9;
    uint32_t m0 = 0xD2511F53u, m1 = 0xCD9E8D57u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            uint32_t h0, l0, h1, l1;
            if (SPLIT) {
                h0 = __umulhi(m0, c0); l0 = m0o * c0;
                h1 = __umulhi(m1, c2); l1 = m1o * c2;
            } else {
                uint64_t p0 = (uint64_t)m0 * c0, p1 = (uint64_t)m1 * c2;
                h0 = p0 >> 32; l0 = (uint32_t)p0; h1 = p1 >> 32; l1 = (uint32_t)p1;
            }
            uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
            c0 = n0; c1 = l1; c2 = n2; c3 = l0; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
        }
    }
    if ((c0 ^ c1 ^ c2 ^ c3) == 0x12345678u) out[0] = 1;
}

int main() {
    uint32_t* d; cudaMalloc(&d, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int split = 0; split < 2; ++split) {
        for (int threads : {256, 512, 1024}) {
            int blocks = 148 * (2048 / threads);
            int iters = 2000;
            if (split) k<1><<<blocks, threads>>>(d, 1, 2, 10, 0xD2511F53u, 0xCD9E8D57u); else k<0><<<blocks, threads>>>(d, 1, 2, 10, 0xD2511F53u, 0xCD9E8D57u);
            cudaEventRecord(a);
            if (split) k<1><<<blocks, threads>>>(d, 1, 2, iters, 0xD2511F53u, 0xCD9E8D57u); else k<0><<<blocks, threads>>>(d, 1, 2, iters, 0xD2511F53u, 0xCD9E8D57u);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double rounds = (double)blocks * threads * iters * 10;
            printf("split=%d threads=%d: %.3f ms, %.1f G philox-rounds/s\n", split, threads, ms, rounds / ms / 1e6);
        }
    }
}
