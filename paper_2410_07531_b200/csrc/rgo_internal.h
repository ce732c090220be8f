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

// Vector (128-element unit) index map of a row window: compact chunk vector v ->
// vector of the full layout.  wv = vectors per slice window, sv = per slice,
// ov = vector offset of the window's first row.  wv == 0: identity.
struct VecWindow {
    uint64_t wv = 0, sv = 0, ov = 0;
};
__host__ __device__ inline uint64_t window_vec(const VecWindow& w, uint64_t v) {
    if (w.wv == 0) return v;
    const uint64_t s = v < 0xFFFFFFFFull && w.wv <= 0xFFFFFFFFull
                           ? static_cast<uint64_t>(static_cast<uint32_t>(v) / static_cast<uint32_t>(w.wv))
                           : v / w.wv;
    return s * w.sv + w.ov + (v - s * w.wv);
}
// One dropout-mask generation job in the reference layout (mask.hpp:24-48).
struct MaskJob {
    uint8_t* out;           // packed bits, 16-byte aligned
    uint64_t elems;         // B*nH*SQ^2
    uint64_t seed;
    uint64_t base_offset;
    uint64_t threshold;     // KeepThreshold::threshold(), in [0, 2^32]
    int rounds;             // [1,16]
    // Row window (SQ-chunk pipelining, schedule.hpp:205-239): when win_rows > 0,
    // `elems` = slices * win_rows * seq and out holds the compact chunk mask
    // [slice][win_rows][seq] of rows [row0, row0 + win_rows) of every slice of a
    // layout with `seq` rows/keys: element (s, i, j) takes the keep bit of the
    // full layout's element (s*seq + row0 + i)*seq + j.  Needs seq % 128 == 0.
    uint32_t win_rows = 0, row0 = 0, seq = 0;
    // General vector window (wv > 0 overrides the row window): out holds the compact
    // mask of the layout's vectors window_vec(vwin, v) -- e.g. a tensor-parallel
    // rank's heads [h0, h0+Hl) of every batch item (wv = Hl*SQ^2/128, sv = nH*SQ^2/128,
    // ov = h0*SQ^2/128, capacity.hpp:14-26), counters of the full layout.
    VecWindow vwin{};
};

inline VecWindow make_window(uint32_t win_rows, uint32_t row0, uint32_t seq) {
    VecWindow w;
    if (win_rows == 0) return w;
    w.wv = static_cast<uint64_t>(win_rows) * seq / 128;
    w.sv = static_cast<uint64_t>(seq) * seq / 128;
    w.ov = static_cast<uint64_t>(row0) * seq / 128;
    return w;
}

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

// Per-device staging workspace of the host-buffer entry points (the drop-in
// forms of the reference's value-semantics API): one grow-only device
// allocation per device, reused across calls instead of cudaMalloc/cudaFree per
// call.  Callers hold `mu` for the whole call (the host entry points are
// synchronous, so the buffer is idle again when they return).
struct HostWorkspace {
    std::mutex mu;
    void* p = nullptr;
    size_t cap = 0;
    // a buffer of >= n bytes (256-byte aligned); call with mu held
    cudaError_t get(size_t n, void** out) {
        if (n > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            const size_t want = n + (n >> 2);  // headroom for slightly larger calls
            cudaError_t e = cudaMalloc(&p, want);
            if (e != cudaSuccess) return e;
            cap = want;
        }
        *out = p;
        return cudaSuccess;
    }
};
HostWorkspace& host_workspace();  // the current device's

int num_sms();
int mask_kernel_occupancy(int rounds, int block, size_t dyn_smem);
cudaError_t launch_mask(const MaskJob& j, const LaunchShape& shape, cudaStream_t s);
cudaError_t launch_philox_blocks(const uint32_t* keys, const uint32_t* ctrs, const int* rounds,
                                 uint32_t* out, uint64_t n, cudaStream_t s);
cudaError_t launch_uniform_bf16(uint64_t seed, uint32_t stream_id, uint64_t n, void* out_bf16,
                                float* out_f32, cudaStream_t s);

}  // namespace rgo
