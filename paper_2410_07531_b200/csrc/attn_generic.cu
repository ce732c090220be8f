// attn_generic.cu -- K5g: attention forward with dropout for any head_dim, fp32.
//
// The drop-in's attention_forward / _dropout_fused / _dropout_decoupled
// (ref_attention.hpp:56-146) accept any head_dim; the tcgen05 kernels (K5/K6,
// attn_fwd_sm100.cu) cover head_dim <= 128 on bf16 operands.  Above that the
// host entry point runs this kernel instead: fp32 operands, fp32 arithmetic
// on the CUDA cores, the reference's semantics (ref_attention.hpp:66-90):
//   w_j = exp(scale * q.k_j - max_j), weight_j = w_j / sum_j w_j (ALL keys),
//   kept weights / p, dropped 0, o = sum_j weight_j v_j,
// with the keep bit of element (s*SQ + i)*SQ + j read from the bitmask
// (decoupled) or regenerated with Philox-R at counter base_offset + idx/4
// (fused, mask.hpp:72-92).  One warp per query row: lanes split the head
// dimension (coalesced K/V rows, butterfly-reduced dot products), online
// softmax in registers, NC = ceil(head_dim / 32) output columns per lane.
#include <cuda_runtime.h>

#include <cstdint>

#include "attn.h"
#include "philox.cuh"

namespace rgo_attn_generic {

struct Params {
    const float *q, *k, *v;
    float* o;
    uint32_t slices, S, HD;
    float scale, keep_prob;
    int mode;  // MASK_NONE / MASK_BITS / MASK_PHILOX
    const uint8_t* bits;
    uint32_t k0, k1, thr;
    uint64_t base_offset;
    int rounds;
};

template <int NC>
__global__ void __launch_bounds__(256) attn_generic_kernel(const Params p) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t row = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // slice * S + i
    if (row >= static_cast<uint64_t>(p.slices) * p.S) return;
    const uint64_t slice = row / p.S;
    const float* qr = p.q + row * p.HD;
    const float* kb = p.k + slice * p.S * p.HD;
    const float* vb = p.v + slice * p.S * p.HD;
    float qv[NC], o[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint32_t d = lane + 32u * c;
        qv[c] = d < p.HD ? qr[d] : 0.0f;
        o[c] = 0.0f;
    }
    float m = -INFINITY, l = 0.0f;
    for (uint32_t j = 0; j < p.S; ++j) {
        const float* kr = kb + static_cast<uint64_t>(j) * p.HD;
        float dot = 0.0f;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const uint32_t d = lane + 32u * c;
            if (d < p.HD) dot = fmaf(qv[c], kr[d], dot);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        const float sc = dot * p.scale;  // identical in every lane (butterfly)
        if (sc > m) {
            const float alpha = __expf(m - sc);  // 0 on the first key
#pragma unroll
            for (int c = 0; c < NC; ++c) o[c] *= alpha;
            l *= alpha;
            m = sc;
        }
        const float w = expf(sc - m);
        l += w;  // the denominator sums every key, before dropout (ref_attention.hpp:78-82)
        bool keep = true;
        if (p.mode != rgo_attn::MASK_NONE) {
            const uint64_t idx = row * p.S + j;
            if (p.mode == rgo_attn::MASK_BITS) {
                keep = (p.bits[idx >> 3] >> (idx & 7)) & 1u;
            } else {
                const uint64_t ctr = p.base_offset + (idx >> 2);
                const uint4 r = rgo_dev::philox_rt(static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), 0u,
                                                   0u, p.k0, p.k1, p.rounds);
                const uint32_t e = static_cast<uint32_t>(idx & 3);
                keep = (e == 0 ? r.x : e == 1 ? r.y : e == 2 ? r.z : r.w) < p.thr;
            }
        }
        if (keep) {
            const float* vr = vb + static_cast<uint64_t>(j) * p.HD;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const uint32_t d = lane + 32u * c;
                if (d < p.HD) o[c] = fmaf(w, vr[d], o[c]);
            }
        }
    }
    const float inv = 1.0f / (l * p.keep_prob);
    float* orow = p.o + row * p.HD;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint32_t d = lane + 32u * c;
        if (d < p.HD) orow[d] = o[c] * inv;
    }
}

}  // namespace rgo_attn_generic

namespace rgo {

cudaError_t launch_attn_generic_f32(const float* q, const float* k, const float* v, float* o, uint32_t slices,
                                    uint32_t S, uint32_t HD, float scale, int mode, float keep_prob,
                                    const uint8_t* bits, uint64_t seed, uint64_t threshold, uint64_t base_offset,
                                    int rounds, cudaStream_t s) {
    using namespace rgo_attn_generic;
    using rgo_attn::MASK_NONE;
    using rgo_attn::MASK_PHILOX;
    if (HD == 0 || HD > kGenericMaxHeadDim) return cudaErrorInvalidValue;
    Params p{};
    p.q = q; p.k = k; p.v = v; p.o = o;
    p.slices = slices; p.S = S; p.HD = HD;
    p.scale = scale;
    p.mode = mode;
    // keep-all threshold (2^32): every bit is 1 -> no dropout test, still scaled by 1/p
    if (mode == MASK_PHILOX && threshold >= (uint64_t{1} << 32)) p.mode = MASK_NONE;
    p.keep_prob = mode == MASK_NONE ? 1.0f : keep_prob;
    p.bits = bits;
    p.k0 = static_cast<uint32_t>(seed);
    p.k1 = static_cast<uint32_t>(seed >> 32);
    p.thr = static_cast<uint32_t>(threshold);
    p.base_offset = base_offset;
    p.rounds = rounds;
    const uint64_t warps = static_cast<uint64_t>(slices) * S;
    const dim3 grid(static_cast<unsigned>((warps * 32 + 255) / 256));
    const uint32_t nc = (HD + 31) / 32;
    if (nc <= 8)
        attn_generic_kernel<8><<<grid, 256, 0, s>>>(p);
    else if (nc <= 16)
        attn_generic_kernel<16><<<grid, 256, 0, s>>>(p);
    else
        attn_generic_kernel<32><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace rgo
