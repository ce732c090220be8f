// Microbenchmark: TMA bulk reduce-add (fp32) throughput from smem to global,
// vs REDG.v4 from registers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_red.cu -o bulk_red
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void bulk_kernel(float* dst, size_t region_floats, int iters, int chunk_bytes, int inflight) {
    extern __shared__ __align__(128) uint8_t sm[];
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        float* base = dst + (size_t)blockIdx.x * region_floats;
        size_t off = 0;
        uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
        for (int it = 0; it < iters; ++it) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(base + off),
                         "r"(s + (it % 2) * 32768 % 65536), "r"(chunk_bytes) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (inflight == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else if (inflight == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
            off += chunk_bytes / 4;
            if (off + chunk_bytes / 4 > region_floats) off = 0;
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void redg_kernel(float* dst, size_t region_floats, int iters) {
    float* base = dst + (size_t)blockIdx.x * region_floats;
    size_t off = 0;
    for (int it = 0; it < iters; ++it) {
        float* p = base + off + threadIdx.x * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
        off += blockDim.x * 4;
        if (off + blockDim.x * 4 > region_floats) off = 0;
    }
}

int main() {
    int sms = 148;
    float* d;
    size_t total = (size_t)1 << 30;  // 4 GB of floats? no: 1 Gi floats = 4 GB
    cudaMalloc(&d, total * 4);
    cudaMemset(d, 0, total * 4);
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (size_t region_kb : {64, 512, 2048, 16384}) {
        for (int chunk : {4096, 16384, 32768}) {
            for (int inflight : {1, 2, 4}) {
                size_t region = region_kb * 256;
                int iters = 2000;
                bulk_kernel<<<sms, 128, 65536>>>(d, region, 10, chunk, inflight);
                cudaEventRecord(a);
                bulk_kernel<<<sms, 128, 65536>>>(d, region, iters, chunk, inflight);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                double bytes = (double)sms * iters * chunk;
                printf("bulk region/CTA %6zu KB chunk %6d inflight %d: %.2f TB/s\n", region_kb, chunk, inflight, bytes / ms / 1e9);
            }
        }
        for (int threads : {128, 512}) {
            size_t region = region_kb * 256;
            int iters = 4000;
            redg_kernel<<<sms * 2, threads>>>(d, region, 10);
            cudaEventRecord(a);
            redg_kernel<<<sms * 2, threads>>>(d, region, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double bytes = (double)sms * 2 * iters * threads * 16;
            printf("redg region/CTA %6zu KB threads %d: %.2f TB/s\n", region_kb, threads, bytes / ms / 1e9);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
