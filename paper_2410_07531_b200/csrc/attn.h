// attn.h -- internal attention launch interface.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rgo_attn {
enum { MASK_NONE = 0, MASK_BITS = 1, MASK_PHILOX = 2 };

struct AttnParams {
    int B, H, S;             // S = keys per slice (the layout's SQ)
    int Sq;                  // query rows of this launch per slice (S, or a pipeline chunk's rows)
    int q_row0;              // global row of query 0 (mask counters, LSE): 0, or the chunk's first row
    int bits_rows;           // MASK_BITS: rows per slice in `bits` (S: full layout; Sq: a chunk's mask)
    int n_pairs;             // ceil(Sq / 256): CTAs per (b, h)
    float scale_log2;        // log2(e) / sqrt(head_dim)
    float keep_prob;         // float keep probability (1 for no dropout)
    const uint8_t* bits;     // MASK_BITS: packed mask, reference layout
    uint64_t bits_bytes;
    int bits_aligned;        // SQ % 128 == 0 and 16-byte aligned bits
    int mask_tma;            // MASK_BITS: keep-bit tiles arrive by TMA (bits_aligned, the kernel's tmM)
    int o_tma;               // O leaves by TMA store (the kernel's tmO)
    int resident;            // CTAs resident at once (SMs): the Q prefetch's next CTA = blockIdx + resident
    uint32_t k0, k1;         // MASK_PHILOX: key
    uint64_t base_offset;
    uint32_t thr;            // threshold < 2^32
    int rounds;
    void* O;                 // bf16 output rows
    long long o_sb, o_sh, o_ss;  // element strides of batch, head, position
    float* lse;              // natural-log LSE per (slice, row), or null
    int Hg, h0;              // MASK_PHILOX global slice = b*Hg + h0 + h (AttnJob::Hg)
};

#ifdef __CUDACC__
// Dropout on a packed bf16 pair: given ksh[t] = kw << t (kw: 32 keep bits,
// LSB first), returns the half-word mask (0x0000 / 0xFFFF per half) of keep
// bits (e, e+1), e even.  kw << t puts bit 8b+7-t at the msb of byte b, so
// PRMT's sign-replicate selectors pick bit e from one shifted copy and bit
// e+1 from the next: one PRMT per pair (plus 7 shifts per 32 keys) instead
// of a bit test + select per element; the caller ANDs it into the pair.
__device__ __forceinline__ uint32_t keep_pair_mask(const uint32_t (&ksh)[8], int e) {
    constexpr uint32_t kSel[4] = {0xCC88u, 0xDD99u, 0xEEAAu, 0xFFBBu};
    const int pos = e & 7;
    uint32_t m;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(m) : "r"(ksh[7 - pos]), "r"(ksh[6 - pos]), "r"(kSel[e >> 3]));
    return m;
}
#endif
}  // namespace rgo_attn

namespace rgo {

// A bf16 [B, nH, S, HD] view with arbitrary (batch, head, position) strides in
// elements; the head dimension is contiguous.  Covers both the reference
// layout (slice-major, ref_attention.hpp:20-31) and the token-major QKV GEMM
// output ([B*S, 3*H] with a column offset per Q/K/V).
struct AttnTensor {
    const void* ptr;
    long long sb, sh, ss;
};
struct AttnOut {
    void* ptr;
    long long sb, sh, ss;
};

struct AttnJob {
    int B, H, S, HD;         // HD in {64, 128}
    // Query-row window (SQ-chunk pipelining, schedule.hpp:205-239): rows
    // [q_row0, q_row0 + Sq) of every slice attend over all S keys; q and o
    // point at row q_row0.  Sq = 0 means the whole sequence.  bits_rows: rows
    // per slice held in `bits` (0 = S: the full layout, read at row q_row0;
    // Sq: a compact chunk mask [slice][Sq][S]).  Keep bits / Philox counters
    // are the full layout's: element (s*S + q_row0 + i)*S + j.
    int Sq, q_row0, bits_rows;
    float scale;             // 1/sqrt(true head_dim)
    AttnTensor q, k, v;
    AttnOut o;
    float* lse;
    int mode;                // rgo_attn::MASK_*
    float keep_prob;
    const uint8_t* bits;
    uint64_t bits_bytes;
    uint64_t seed, base_offset, threshold;
    int rounds;
    bool pdl;                // programmatic dependent launch after the previous kernel in the stream
    // Tensor-parallel head window: the launch's H heads are heads [h0, h0 + H) of a
    // layout with Hg heads per batch item (Hg = 0: the launch's own layout).  Philox
    // counters (MASK_PHILOX) are the global layout's, slice b*Hg + h0 + h; the bits
    // (MASK_BITS) are the rank's compact mask, slice b*H + h.
    int Hg = 0, h0 = 0;
};

cudaError_t launch_attn_fwd(const AttnJob& j, cudaStream_t s);

// K5g (attn_generic.cu): fp32 CUDA-core forward for head_dim in (128, 1024]
// -- the drop-in's head dims the tcgen05 kernels do not cover.  q/k/v/o are
// the reference's slice-major fp32 arrays ([slices][S][HD]); same mask sources
// and semantics as launch_attn_fwd.
constexpr uint32_t kGenericMaxHeadDim = 1024;
cudaError_t launch_attn_generic_f32(const float* q, const float* k, const float* v, float* o, uint32_t slices,
                                    uint32_t S, uint32_t HD, float scale, int mode, float keep_prob,
                                    const uint8_t* bits, uint64_t seed, uint64_t threshold, uint64_t base_offset,
                                    int rounds, cudaStream_t s);

// K7 backward (attn_bwd_sm100.cu): dQ, dK, dV from Q, K, V, the forward
// output O, its natural-log LSE and dO; same mask sources as the forward.
struct AttnBwdJob {
    int B, H, S, HD;
    float scale;
    AttnTensor q, k, v, o, dout;
    AttnOut dq, dk, dv;
    const float* lse;        // [B*H*S] from the forward
    int mode;                // rgo_attn::MASK_*
    float keep_prob;
    const uint8_t* bits;
    uint64_t bits_bytes;
    uint64_t seed, base_offset, threshold;
    int rounds;
    void* work;              // attn_bwd_workspace_bytes()
    bool deterministic;      // head_dim 128: split backward, dQ in TMEM (no cross-CTA reductions)
};

uint64_t attn_bwd_workspace_bytes(int B, int H, int S, int HD);
cudaError_t launch_attn_bwd(const AttnBwdJob& j, cudaStream_t s);

}  // namespace rgo
