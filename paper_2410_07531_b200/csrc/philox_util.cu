// philox_util.cu -- device Philox utilities used by the C ABI:
//  * philox_blocks_kernel: philox_block over arrays of (key, counter, rounds);
//    lets the GPU path be checked against the reference KATs and the
//    random-vector suites (test_philox.cpp:78-111, acceptance_main.cpp:75-97).
//  * uniform_kernel: random_attention_input's generator
//    (ref_attention.hpp:186-202) on device: Philox-10, counter
//    (block lo, block hi, stream, 0x5eed), value = float(w)*(2/2^32) - 1
//    computed with explicit round-to-nearest intrinsics so no FMA contraction
//    can change it; optionally rounded to bf16 for the tensor-core kernels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "philox.cuh"
#include "rgo_internal.h"

namespace rgo_dev {

__global__ void philox_blocks_kernel(const uint32_t* __restrict__ keys,
                                     const uint32_t* __restrict__ ctrs,
                                     const int* __restrict__ rounds, uint32_t* __restrict__ out,
                                     uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 w = philox_rt(ctrs[4 * i], ctrs[4 * i + 1], ctrs[4 * i + 2], ctrs[4 * i + 3],
                              keys[2 * i], keys[2 * i + 1], rounds[i]);
    out[4 * i] = w.x;
    out[4 * i + 1] = w.y;
    out[4 * i + 2] = w.z;
    out[4 * i + 3] = w.w;
}

__global__ void uniform_kernel(uint64_t seed, uint32_t stream_id, uint64_t n,
                               __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_f32) {
    const uint64_t blk = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t i = blk * 4;
    if (i >= n) return;
    const uint4 w = philox<10>(static_cast<uint32_t>(blk), static_cast<uint32_t>(blk >> 32),
                               stream_id, 0x5eedu, static_cast<uint32_t>(seed),
                               static_cast<uint32_t>(seed >> 32));
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        if (i + l >= n) break;
        const float f = __fsub_rn(__fmul_rn(__uint2float_rn(ws[l]), 2.0f / 4294967296.0f), 1.0f);
        if (out_f32) out_f32[i + l] = f;
        if (out_bf16) out_bf16[i + l] = __float2bfloat16_rn(f);
    }
}

}  // namespace rgo_dev

namespace rgo {

cudaError_t launch_philox_blocks(const uint32_t* keys, const uint32_t* ctrs, const int* rounds,
                                 uint32_t* out, uint64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    rgo_dev::philox_blocks_kernel<<<grid, 256, 0, s>>>(keys, ctrs, rounds, out, n);
    return cudaGetLastError();
}

cudaError_t launch_uniform_bf16(uint64_t seed, uint32_t stream_id, uint64_t n, void* out_bf16,
                                float* out_f32, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 3) / 4;
    const unsigned grid = static_cast<unsigned>((blocks + 255) / 256);
    rgo_dev::uniform_kernel<<<grid, 256, 0, s>>>(seed, stream_id, n,
                                                 static_cast<__nv_bfloat16*>(out_bf16), out_f32);
    return cudaGetLastError();
}

}  // namespace rgo
