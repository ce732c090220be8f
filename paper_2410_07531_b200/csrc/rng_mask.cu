// rng_mask.cu -- K1: stand-alone Philox dropout-mask kernel (sm_100a).
//
// Replaces mask_detail::fill_byte_range / generate_mask
// (proj/include/rgo/mask.hpp:111-179).  Layout is the reference's:
// element e (global linear index ((b*nH+h)*SQ+i)*SQ+j, mask.hpp:35-39) takes
// lane e&3 of philox_block(seed, ctr = base_offset + (e>>2)) (mask.hpp:72-85)
// and is kept iff word < threshold (mask.hpp:67); bits are packed LSB-first,
// bit e&7 of byte e>>3 (mask.hpp:101-104, 130).
//
// Work unit = one 16-byte vector = 128 elements = 32 Philox blocks; one
// thread builds it in registers and writes it with one st.global.v4, so a
// warp writes 512 contiguous bytes.  The kernel is integer-issue bound
// (R+2 ops/element); the 1-bit output is 1/32 of a 32-bit word per element,
// so HBM is never the limiter.  Grid is persistent (grid-stride), sized as a
// multiple of the SM count, or capped by the caller so it can co-reside with a
// GEMM on the other stream (overlap mechanism A).
#include <cuda_runtime.h>

#include <cstdint>

#include "philox.cuh"
#include "rgo_internal.h"

namespace rgo_dev {

__device__ __forceinline__ void st_v4_streaming(uint8_t* p, uint32_t a, uint32_t b, uint32_t c,
                                                uint32_t d) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

// Vectors [0, n_vec) of the mask; vector v covers elements [128v, 128v+128)
// (WIN: of the row window `win`, written compactly; counters of the full layout).
template <int R, bool WIN>
__global__ void __launch_bounds__(256, (R == 4 || R == 5) ? 4 : 0) rng_mask_kernel(uint8_t* __restrict__ out, uint64_t n_vec,
                                                       uint64_t base_offset, uint32_t k0,
                                                       uint32_t k1, uint32_t thr, uint32_t zero,
                                                       const rgo::VecWindow win) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    // key / threshold in vector registers rather than uniform registers, so a
    // co-resident GEMM keeps the uniform datapath it issues MMAs/TMA through
    asm volatile("" : "+r"(k0), "+r"(k1), "+r"(thr) : "r"(threadIdx.x));
    for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n_vec;
         v += stride) {
        const uint64_t ctr = base_offset + (WIN ? rgo::window_vec(win, v) : v) * 32;  // 64-bit wrap like element_source
        const uint32_t lo = static_cast<uint32_t>(ctr), hi = static_cast<uint32_t>(ctr >> 32);
        uint32_t w0, w1, w2, w3;
        if (lo <= 0xFFFFFFFFu - 31u) {  // no carry into c1 inside this unit
            w0 = keep32_nowrap<R>(lo + 0, hi, k0, k1, thr, zero);
            w1 = keep32_nowrap<R>(lo + 8, hi, k0, k1, thr, zero);
            w2 = keep32_nowrap<R>(lo + 16, hi, k0, k1, thr, zero);
            w3 = keep32_nowrap<R>(lo + 24, hi, k0, k1, thr, zero);
        } else {
            w0 = keep32<R>(ctr + 0, k0, k1, thr);
            w1 = keep32<R>(ctr + 8, k0, k1, thr);
            w2 = keep32<R>(ctr + 16, k0, k1, thr);
            w3 = keep32<R>(ctr + 24, k0, k1, thr);
        }
        st_v4_streaming(out + v * 16, w0, w1, w2, w3);
    }
}

// Tail: elements [128*n_vec, n) (< 128 of them) -> bytes [16*n_vec, nbytes).
// One warp; lane L owns byte 16*n_vec + L (L < 16).  Padding bits stay 0
// (mask.hpp:128 `if (idx >= n) break`).
__global__ void rng_mask_tail_kernel(uint8_t* __restrict__ out, uint64_t n, uint64_t n_vec,
                                     uint64_t base_offset, uint32_t k0, uint32_t k1, uint64_t thr,
                                     int rounds) {
    const uint64_t nbytes = (n + 7) / 8;
    const uint64_t byte = n_vec * 16 + threadIdx.x;
    if (threadIdx.x >= 16 || byte >= nbytes) return;
    uint32_t acc = 0;
    for (int half = 0; half < 2; ++half) {
        const uint64_t block = byte * 2 + half;
        if (block * 4 >= n) break;
        const uint64_t c = base_offset + block;
        const uint4 w =
            philox_rt(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32), 0u, 0u, k0, k1, rounds);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        for (int lane = 0; lane < 4; ++lane) {
            const uint64_t idx = block * 4 + lane;
            if (idx >= n) break;
            if (static_cast<uint64_t>(ws[lane]) < thr) acc |= 1u << (idx & 7);
        }
    }
    out[byte] = static_cast<uint8_t>(acc);
}

// threshold == 0 (keep nothing) or 2^32 (keep everything): every word
// compares the same way, so the mask is constant; padding bits stay 0.
__global__ void mask_fill_kernel(uint8_t* __restrict__ out, uint64_t n, uint8_t value) {
    const uint64_t nbytes = (n + 7) / 8;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nbytes;
         i += stride) {
        uint8_t b = value;
        if (i == nbytes - 1 && (n & 7)) b &= static_cast<uint8_t>((1u << (n & 7)) - 1);
        out[i] = b;
    }
}

// Generic R in [1,16] via a switch over template instances.
// The mask kernels use no shared memory, but an SM's L1/shared split is chosen
// when CTAs are placed and cannot change while any CTA is resident: a kernel
// that lets the driver pick a small carveout would lock a concurrently
// launched GEMM / attention CTA (~200 KB smem) out of every SM it occupies,
// serialising the "overlap".  Preferring the maximum carveout keeps the SMs
// configured for the tensor-core kernels, so the two really co-reside.
template <typename K>
static void prefer_max_smem(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
}

template <int R>
static cudaError_t launch_r(uint8_t* out, uint64_t n_vec, uint64_t base, uint32_t k0, uint32_t k1,
                            uint32_t thr, const rgo::LaunchShape& ls, const rgo::VecWindow& win, cudaStream_t s) {
    static bool once = (prefer_max_smem(rng_mask_kernel<R, false>), prefer_max_smem(rng_mask_kernel<R, true>), true);
    (void)once;
    if (win.wv)
        rng_mask_kernel<R, true><<<ls.grid, ls.block, ls.dyn_smem, s>>>(out, n_vec, base, k0, k1, thr, 0u, win);
    else
        rng_mask_kernel<R, false><<<ls.grid, ls.block, ls.dyn_smem, s>>>(out, n_vec, base, k0, k1, thr, 0u, win);
    return cudaGetLastError();
}

static const void* kernel_ptr(int rounds) {
    switch (rounds) {
#define RGO_CASE(R) \
    case R:         \
        return reinterpret_cast<const void*>(&rng_mask_kernel<R, false>);
        RGO_CASE(1) RGO_CASE(2) RGO_CASE(3) RGO_CASE(4) RGO_CASE(5) RGO_CASE(6) RGO_CASE(7)
        RGO_CASE(8) RGO_CASE(9) RGO_CASE(10) RGO_CASE(11) RGO_CASE(12) RGO_CASE(13)
        RGO_CASE(14) RGO_CASE(15) RGO_CASE(16)
#undef RGO_CASE
        default:
            return nullptr;
    }
}

static const void* kernel_ptr_win(int rounds) {
    switch (rounds) {
#define RGO_CASE(R) \
    case R:         \
        return reinterpret_cast<const void*>(&rng_mask_kernel<R, true>);
        RGO_CASE(1) RGO_CASE(2) RGO_CASE(3) RGO_CASE(4) RGO_CASE(5) RGO_CASE(6) RGO_CASE(7)
        RGO_CASE(8) RGO_CASE(9) RGO_CASE(10) RGO_CASE(11) RGO_CASE(12) RGO_CASE(13)
        RGO_CASE(14) RGO_CASE(15) RGO_CASE(16)
#undef RGO_CASE
        default:
            return nullptr;
    }
}

}  // namespace rgo_dev

namespace rgo {

// Occupancy of the mask kernel at the requested dynamic smem (used to size
// a persistent grid; the dyn_smem knob throttles CTAs/SM for co-residency).
int mask_kernel_occupancy(int rounds, int block, size_t dyn_smem) {
    const void* k = rgo_dev::kernel_ptr(rounds);
    if (!k) return 0;
    if (dyn_smem > 48 * 1024)
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(dyn_smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, block, dyn_smem) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_mask(const MaskJob& j, const LaunchShape& shape_in, cudaStream_t s) {
    using namespace rgo_dev;
    const uint64_t n = j.elems;
    const uint32_t k0 = static_cast<uint32_t>(j.seed), k1 = static_cast<uint32_t>(j.seed >> 32);
    if (j.threshold == 0 || j.threshold >= (uint64_t{1} << 32)) {
        const uint64_t nbytes = (n + 7) / 8;
        const uint64_t blocks = (nbytes + 255) / 256;
        const unsigned grid = static_cast<unsigned>(blocks < 148 * 8 ? blocks : 148 * 8);
        static bool once = (prefer_max_smem(mask_fill_kernel), true);
        (void)once;
        mask_fill_kernel<<<grid, 256, 0, s>>>(j.out, n, j.threshold ? 0xFF : 0x00);
        return cudaGetLastError();
    }
    const uint32_t thr = static_cast<uint32_t>(j.threshold);
    const uint64_t n_vec = n / 128;
    const VecWindow win = j.vwin.wv ? j.vwin : make_window(j.win_rows, j.row0, j.seq);
    if (j.win_rows && (j.seq % 128 || n % 128)) return cudaErrorInvalidValue;
    if (j.vwin.wv && n % 128) return cudaErrorInvalidValue;
    if (n_vec > 0) {
        LaunchShape ls = shape_in;
        if (ls.block == 0) ls.block = 256;
        if (ls.grid == 0) {
            int occ = mask_kernel_occupancy(j.rounds, static_cast<int>(ls.block), ls.dyn_smem);
            if (occ <= 0) occ = 1;
            const uint64_t want = (n_vec + ls.block - 1) / ls.block;
            const uint64_t cap = static_cast<uint64_t>(num_sms()) * occ;
            ls.grid = static_cast<unsigned>(want < cap ? want : cap);
        }
        if (ls.dyn_smem > 48 * 1024) {
            cudaFuncSetAttribute(kernel_ptr(j.rounds), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(ls.dyn_smem));
            cudaFuncSetAttribute(kernel_ptr_win(j.rounds), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(ls.dyn_smem));
        }
        cudaError_t e;
        switch (j.rounds) {
#define RGO_CASE(R)                                                     \
    case R:                                                             \
        e = launch_r<R>(j.out, n_vec, j.base_offset, k0, k1, thr, ls, win, s); \
        break;
            RGO_CASE(1) RGO_CASE(2) RGO_CASE(3) RGO_CASE(4) RGO_CASE(5) RGO_CASE(6) RGO_CASE(7)
            RGO_CASE(8) RGO_CASE(9) RGO_CASE(10) RGO_CASE(11) RGO_CASE(12) RGO_CASE(13)
            RGO_CASE(14) RGO_CASE(15) RGO_CASE(16)
#undef RGO_CASE
            default:
                return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
    }
    if (n % 128) {
        rng_mask_tail_kernel<<<1, 32, 0, s>>>(j.out, n, n_vec, j.base_offset, k0, k1, j.threshold,
                                              j.rounds);
        return cudaGetLastError();
    }
    return cudaSuccess;
}

}  // namespace rgo

// ------------------------------------------------------------------------
// Queue kernel: drains the shared dropout-mask work queue (rng_queue.cuh).
// Used as the tail after GEMM-resident RNG warps (mechanism B) and as a
// dynamically scheduled stand-alone generator.
#include "rng_queue.cuh"

namespace rgo_dev {
template <int R>
__global__ void __launch_bounds__(256) rng_queue_kernel(const rgo::RngQueue q) {
    // As a programmatic dependent (block tail after the last GEMM): start draining
    // while the GEMM's last CTAs finish, let the attention kernel launch early, and
    // complete only after the GEMM has (so the attention sees the GEMM's output).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    rgo::rng_drain_r<R>(q, nullptr, 0);
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
}  // namespace rgo_dev

namespace rgo {
cudaError_t launch_rng_queue(const RngQueue& q, unsigned grid, unsigned block, size_t dyn_smem,
                             cudaStream_t s, bool pdl) {
    if (block == 0) block = 256;
    if (grid == 0) grid = static_cast<unsigned>(num_sms()) * 3;
    switch (q.rounds) {
#define RGO_CASE(R)                                                                  \
    case R:                                                                          \
        if (dyn_smem > 48 * 1024)                                                    \
            cudaFuncSetAttribute(rgo_dev::rng_queue_kernel<R>,                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                 static_cast<int>(dyn_smem));                        \
        cudaFuncSetAttribute(rgo_dev::rng_queue_kernel<R>,                           \
                             cudaFuncAttributePreferredSharedMemoryCarveout,         \
                             cudaSharedmemCarveoutMaxShared);                        \
        {                                                                            \
            cudaLaunchConfig_t cfg{};                                                \
            cudaLaunchAttribute at[1];                                               \
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;           \
            at[0].val.programmaticStreamSerializationAllowed = 1;                    \
            cfg.gridDim = dim3(grid);                                                \
            cfg.blockDim = dim3(block);                                              \
            cfg.dynamicSmemBytes = dyn_smem;                                         \
            cfg.stream = s;                                                          \
            cfg.attrs = at;                                                          \
            cfg.numAttrs = pdl ? 1 : 0;                                              \
            cudaError_t le = cudaLaunchKernelEx(&cfg, rgo_dev::rng_queue_kernel<R>, q); \
            if (le != cudaSuccess) return le;                                        \
        }                                                                            \
        break;
        RGO_CASE(1) RGO_CASE(2) RGO_CASE(3) RGO_CASE(4) RGO_CASE(5) RGO_CASE(6) RGO_CASE(7)
        RGO_CASE(8) RGO_CASE(9) RGO_CASE(10) RGO_CASE(11) RGO_CASE(12) RGO_CASE(13)
        RGO_CASE(14) RGO_CASE(15) RGO_CASE(16)
#undef RGO_CASE
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
}  // namespace rgo
