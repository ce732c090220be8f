// block.h -- internal transformer-block runtime interface (see block.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rgo {

enum { BLOCK_SERIAL_FUSED = 0, BLOCK_STREAMS = 1, BLOCK_IN_GEMM = 2, BLOCK_NO_RNG = 3 };

struct BlockConfig {
    int batch, seq, heads, head_dim, ffn;
    int gated;                   // SwiGLU FFN1 (2*ffn outputs) else GELU
    float keep_prob;             // float keep probability
    uint64_t threshold;          // KeepThreshold::threshold(), < 2^32
    int rounds;
    uint64_t seed, base_offset;  // mask layout (batch*heads slices)
    // per-tensor FP8 scales: alpha = dequant of A.B, s_* = output quantisation
    float a_qkv, a_proj, a_ffn1, a_ffn2;
    float s_attn, s_proj, s_ffn1, s_ffn2;
    // mechanism A launch shape of the mask kernel (0 = auto)
    unsigned rng_grid, rng_block, rng_smem;
    // MoE FFN (experts > 0): `experts` expert FFNs of width ffn, top_k experts
    // per token, balanced synthetic routing (see moe_slot)
    int experts, top_k;
    // SQ-chunk pipelining (schedule.hpp:205-239): chunks > 1 splits the query
    // rows of every sequence into `chunks` windows of seq/chunks rows; the step
    // becomes C stages [attention(c) -> Proj/FFN/QKV of window c] with the RNG
    // of window c+1 hidden under stage c's GEMMs, and the live mask is a 2-slot
    // ring of window masks (2/C of the full mask)
    int chunks;
    // Tensor parallelism (Megatron, capacity.hpp:14-26): tp_size ranks
    // split the heads (QKV and FFN1 column-parallel, Proj and FFN2 row-parallel).  Rank
    // tp_rank owns heads [tp_rank*H/tp, ...) of every batch item, their compact mask
    // (the global layout's keep bits and counters) and an F/tp slice of the FFN; the
    // Proj and FFN2 partial sums are all-reduced over peer memory (two-shot: each rank
    // reduces its M/tp rows of every rank's bf16 partial and quantises them to e4m3,
    // then gathers the other ranks' rows).  heads/ffn/weights/buffers are the rank's.
    int tp_size = 1, tp_rank = 0;
};

struct BlockBuffers {
    void* x;        // e4m3 [M, d]   block input (= FFN2 output of the previous block)
    void* wqkv;     // e4m3 [3d, d]
    void* wo;       // e4m3 [d, d]
    void* w1;       // e4m3 [n1, d]  (SwiGLU: per 256-row tile [128 gate | 128 up])
    void* w2;       // e4m3 [d, ffn]
    void* qkv;      // bf16 [M, 3d]
    void* attn_o;   // bf16 [M, d]
    void* attn_o8;  // e4m3 [M, d]
    void* y1;       // e4m3 [M, d]
    void* h;        // e4m3 [M, ffn]
    uint8_t* mask;  // packed dropout mask, B*nH*S^2/8 bytes
    uint64_t mask_bytes;
    unsigned long long* counter;  // mask work-queue counter (IN_GEMM)
    float* lse;     // optional [B*nH*S]
    void* xd;       // MoE: e4m3 [M*top_k, d] expert-sorted (dispatched) FFN inputs
    void* ye;       // MoE: bf16 [M*top_k, d] expert FFN outputs before the combine
    const void* attn_in;  // bf16 [M, d] step input (previous block's attention output);
                          // null: attn_o, i.e. each step consumes the previous step's output
    void* qkv_out;  // chunked: bf16 [M, 3d] the step's QKV GEMM output (the step's attention
                    // reads qkv, written by the previous step); counter then has chunks entries
    // tensor parallel (tp_size > 1): every rank's bf16 [M, d] partial-sum buffer and
    // its y1 / x (e4m3 [M, d], full d) as mapped in this process ([tp_rank] = own)
    static constexpr int MAX_TP = 8;
    void* peer_part[MAX_TP] = {};
    void* peer_y1[MAX_TP] = {};
    void* peer_x[MAX_TP] = {};
};

// Host-side barrier across the tensor-parallel ranks (called between the step's
// segments, after the rank's stream is synchronised).
typedef void (*TpBarrier)(void* ctx);

struct Block;
cudaError_t block_create(const BlockConfig& cfg, const BlockBuffers& buf, int mode, bool use_graph, Block** out);
cudaError_t block_step(Block* b, cudaStream_t stream, int* launches);
// Tensor-parallel step (tp_size > 1): five segments separated by barrier(ctx) --
// quant + Proj | reduce(Proj) | gather + FFN1 + FFN2 | reduce(FFN2) | gather + QKV +
// attention.  Every rank must call it once per step.
cudaError_t block_step_tp(Block* b, cudaStream_t stream, TpBarrier barrier, void* ctx, int* launches);
int block_tp_size(const Block* b);
// Device time of the last step's phases: [0] GEMM window (quant + 4 GEMMs),
// [1] attention (incl. the RNG join / tail), in ms.
cudaError_t block_last_timings(Block* b, float* ms2);
// [0] GEMM window, [1] RNG tail / join before the attention, [2] attention kernel.
cudaError_t block_last_timings3(Block* b, float* ms3);
void block_destroy(Block* b);
cudaError_t launch_quant_e4m3(const void* in, void* out, uint64_t n, float scale, cudaStream_t s);
// Rows r < rows of [*, d] bf16 -> e4m3, row r at (r / rb) * rstride + roff + r % rb.
cudaError_t launch_quant_e4m3_rows(const void* in, void* out, int rows, int d, int rb, int rstride, int roff,
                                   float scale, cudaStream_t s);

}  // namespace rgo
