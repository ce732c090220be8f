// Diagnostic spin kernels (not part of the product): occupy one pipe for a
// fixed number of iterations so its interference with the tcgen05 GEMM can be
// measured.  mode 0: LOP3/IADD (alu)  1: IMAD.WIDE (fma-heavy)  2: FFMA  3: mask-like mix
#include <cstdint>
#include <cuda_runtime.h>
__global__ void spin(uint32_t* out, int iters, int mode) {
    uint32_t a = threadIdx.x, b = blockIdx.x * 77u + 1u, c = 0x9E3779B9u, d = 12345u;
    uint32_t e = a ^ 0x55u, f = b ^ 0xAAu, g = c ^ 7u, h = d ^ 9u;
    float x = a * 1e-3f, y = b * 1e-3f, z = 1.0001f, w = 0.9999f;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {
#pragma unroll
            for (int k = 0; k < 16; ++k) { a = (a ^ b) + c; b = (b ^ d) + a; e = (e ^ f) + g; f = (f ^ h) + e; }
        } else if (mode == 1) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                uint64_t p = (uint64_t)a * 0xD2511F53u; a = (uint32_t)(p >> 32) ^ b; b = (uint32_t)p;
                uint64_t q = (uint64_t)e * 0xCD9E8D57u; e = (uint32_t)(q >> 32) ^ f; f = (uint32_t)q;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) { x = x * z + w; y = y * w + z; z = z * x + y; w = w * y + x; }
        }
    }
    if (a == 0x12345678u && e == 1u && x == 1.2345f) out[0] = a + b + e + f + __float_as_uint(x + y + z + w);
}
extern "C" int launch_spin(uint32_t* out, int grid, int block, int iters, int mode, void* stream) {
    static bool once = (cudaFuncSetAttribute(spin, cudaFuncAttributePreferredSharedMemoryCarveout, 100), true);
    (void)once;
    spin<<<grid, block, 0, (cudaStream_t)stream>>>(out, iters, mode);
    return (int)cudaGetLastError();
}

// ---- mask-kernel code-footprint variants (diagnostic) ----
#include "../../paper_2410_07531_b200/csrc/philox.cuh"
template <int UNROLL_WORDS>
__global__ void __launch_bounds__(256) mask_var(uint8_t* out, uint64_t n_vec, uint32_t k0, uint32_t k1, uint32_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vec; v += stride) {
        const uint64_t ctr = v * 32;
        const uint32_t lo = (uint32_t)ctr, hi = (uint32_t)(ctr >> 32);
        uint32_t w[4];
        if (UNROLL_WORDS) {
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = rgo_dev::keep32_nowrap<10>(lo + 8 * q, hi, k0, k1, thr, 0u);
        } else {
#pragma unroll 1
            for (int q = 0; q < 4; ++q) w[q] = rgo_dev::keep32_nowrap<10>(lo + 8 * q, hi, k0, k1, thr, 0u);
        }
        *reinterpret_cast<uint4*>(out + v * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}
extern "C" int launch_mask_var(uint8_t* out, uint64_t n_vec, int grid, int block, int unroll, void* stream) {
    static bool once = (cudaFuncSetAttribute(mask_var<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                        cudaFuncSetAttribute(mask_var<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100), true);
    (void)once;
    if (unroll) mask_var<1><<<grid, block, 0, (cudaStream_t)stream>>>(out, n_vec, 1u, 2u, 3865470464u);
    else mask_var<0><<<grid, block, 0, (cudaStream_t)stream>>>(out, n_vec, 1u, 2u, 3865470464u);
    return (int)cudaGetLastError();
}
