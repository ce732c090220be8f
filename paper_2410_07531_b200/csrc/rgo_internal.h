// rgo_internal.h -- internal launch interfaces shared by the .cu units and
// the C ABI (capi.cu).  Not part of the public boundary (include/rgo/capi.h).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

namespace rgo {

struct LaunchShape {
    unsigned grid = 0;      // 0 = auto (persistent, SMs x occupancy)
    unsigned block = 0;     // 0 = kernel default
    size_t dyn_smem = 0;    // extra dynamic smem: throttles CTAs/SM for co-residency
};

// One dropout-mask generation job in the reference layout (mask.hpp:24-48).
struct MaskJob {
    uint8_t* out;           // packed bits, 16-byte aligned
    uint64_t elems;         // B*nH*SQ^2
    uint64_t seed;
    uint64_t base_offset;
    uint64_t threshold;     // KeepThreshold::threshold(), in [0, 2^32]
    int rounds;             // [1,16]
};

// Kernel attributes are per device: set the dynamic shared-memory opt-in once
// per (kernel, current device), so launches on a second GPU of the same
// process do not skip it.  Thread-safe.
inline cudaError_t ensure_dyn_smem(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

int num_sms();
int mask_kernel_occupancy(int rounds, int block, size_t dyn_smem);
cudaError_t launch_mask(const MaskJob& j, const LaunchShape& shape, cudaStream_t s);
cudaError_t launch_philox_blocks(const uint32_t* keys, const uint32_t* ctrs, const int* rounds,
                                 uint32_t* out, uint64_t n, cudaStream_t s);
cudaError_t launch_uniform_bf16(uint64_t seed, uint32_t stream_id, uint64_t n, void* out_bf16,
                                float* out_f32, cudaStream_t s);

}  // namespace rgo
