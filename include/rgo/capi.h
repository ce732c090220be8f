/*
 * rgo/capi.h -- the C-ABI boundary of the B200 dropout-RNG pipeline.
 *
 * The reference (proj/include/rgo/*.hpp) is a header-only C++ library whose
 * entry points are the plugin surface for this path.  Each function below is
 * the device-side replacement for one of them; the C++ headers next to this
 * file (include/rgo/philox.hpp, mask.hpp, ref_attention.hpp, workload.hpp)
 * keep the reference's names and signatures and call through here.
 *
 * Conventions
 *   - plain pointers + byte/element counts; no torch or C++ types;
 *   - device pointers are prefixed d_, host pointers h_;
 *   - rgo_stream_t is a cudaStream_t (NULL = legacy default stream); every
 *     device call is stream-ordered and asynchronous;
 *   - the library never allocates memory that it returns to the caller;
 *   - every call returns an rgo_status; on failure rgo_last_error() returns a
 *     thread-local message (validation messages keep the reference's keywords,
 *     e.g. "bytes"/"guard" for the capacity guard, mask.hpp:148-155);
 *   - there is no CPU fallback: with no CUDA device every compute call fails
 *     with RGO_ENODEV.
 */
#ifndef RGO_CAPI_H
#define RGO_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* rgo_stream_t; /* cudaStream_t */

typedef enum rgo_status {
    RGO_OK = 0,
    RGO_EINVAL = 1,  /* std::invalid_argument in the reference */
    RGO_ECUDA = 2,   /* CUDA runtime / launch failure */
    RGO_ENOMEM = 3,  /* device allocation failed (host wrappers only) */
    RGO_EIO = 4,     /* std::runtime_error in the reference (mask file I/O) */
    RGO_ENODEV = 5   /* no CUDA device: the product has no CPU fallback */
} rgo_status;

const char* rgo_last_error(void);
int rgo_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int rgo_device_count(void);

/* ---------------------------------------------------------------- philox --
 * philox_block(key, counter, rounds) for n independent inputs on device
 * (replaces proj/include/rgo/philox.hpp:84-96).  d_keys: n x {k0,k1},
 * d_ctrs: n x {c0..c3}, d_rounds: n ints in [1,16] (unchecked on device),
 * d_out: n x {w0..w3}. */
int rgo_philox_blocks(const uint32_t* d_keys, const uint32_t* d_ctrs, const int32_t* d_rounds,
                      uint32_t* d_out, uint64_t n, rgo_stream_t stream);

/* ------------------------------------------------------------------ mask --
 * Dropout mask layout (mask.hpp:24-48) + threshold + rounds. */
typedef struct rgo_mask_desc {
    uint32_t batch;
    uint32_t heads;
    uint32_t seq;          /* rows == cols == seq */
    uint32_t rounds;       /* Philox rounds, [1,16] */
    uint64_t seed;         /* key = (seed lo, seed hi), mask.hpp:41-43 */
    uint64_t base_offset;  /* counter of block 0, mask.hpp:28 */
    uint64_t threshold;    /* KeepThreshold::threshold(), [0, 2^32], mask.hpp:62-65 */
} rgo_mask_desc;

/* Launch shaping for the mask kernel (0 = automatic).  grid caps the
 * persistent grid, dyn_smem reserves shared memory per CTA so the kernel only
 * occupies the slots a concurrently running GEMM leaves free. */
typedef struct rgo_launch {
    uint32_t grid;
    uint32_t block;
    uint32_t dyn_smem;
    uint32_t reserved;
} rgo_launch;

/* KeepThreshold(p) (mask.hpp:53-68): keep_prob rounded to float, threshold =
 * llround(double(float p) * 2^32).  RGO_EINVAL unless 0 <= p <= 1. */
int rgo_keep_threshold(double p, uint64_t* threshold, float* keep_prob);

/* ceil(B*nH*SQ^2 / 8); RGO_EINVAL for an empty layout (mask.hpp:45-47). */
int rgo_mask_bytes(const rgo_mask_desc* d, uint64_t* bytes);

/* K1: write the packed keep mask of layout d into d_bits (bytes >=
 * rgo_mask_bytes, 16-byte aligned).  Bit-exact with generate_mask
 * (mask.hpp:142-179) for any layout, threshold and rounds. */
int rgo_mask_generate(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                      rgo_stream_t stream);
int rgo_mask_generate_ex(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                         const rgo_launch* launch, rgo_stream_t stream);

/* Drop-in for generate_mask(layout, thr, rounds, workers): validates like the
 * reference (rounds, empty layout, 2^36-bit guard with a message containing
 * "bytes" and "guard"), generates on `devices` GPUs (0 = all visible; the
 * reference's worker count maps to the device count -- output bytes do not
 * depend on it, mask.hpp:139-141) and copies the bits to h_bits. */
int rgo_generate_mask_host(const rgo_mask_desc* d, uint8_t* h_bits, uint64_t bytes,
                           uint32_t devices);
/* As rgo_generate_mask_host, split into `shards` (>= devices; 0 = one per
 * device) byte-aligned shards, each generated from its own counter offset and
 * copied into place; shard r runs on device (current + r % devices).  The
 * bytes never depend on devices or shards (mask.hpp:139-141); shards > devices
 * exercises the multi-device slicing on one GPU. */
int rgo_generate_mask_host_ex(const rgo_mask_desc* d, uint8_t* h_bits, uint64_t bytes,
                              uint32_t devices, uint32_t shards);

/* ------------------------------------------------------- synthetic inputs --
 * random_attention_input's generator (ref_attention.hpp:186-202) on device:
 * n values uniform in [-1,1) from Philox-10 with counter
 * (i/4 lo, i/4 hi, stream_id, 0x5eed).  Writes fp32 (d_f32, exact) and/or
 * bf16 (d_bf16, round-to-nearest of the fp32 value); either may be NULL. */
int rgo_uniform_fill(uint64_t seed, uint32_t stream_id, uint64_t n, void* d_bf16, float* d_f32,
                     rgo_stream_t stream);

/* Dropout-mask work queue (overlap mechanism B tail / dynamic scheduling):
 * drains vectors [*d_counter, n/128) of layout d into d_bits, claiming
 * 64-vector chunks with atomics on d_counter (zero it before the first
 * producer of a pass).  Requires B*nH*SQ^2 % 128 == 0 and threshold < 2^32. */
int rgo_mask_queue_drain(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                         unsigned long long* d_counter, const rgo_launch* launch,
                         rgo_stream_t stream);

/* ------------------------------------------------------------------ GEMM --
 * K2/K3: C[m, n_out] = epilogue(alpha * A[m,k] . B[n,k]^T) * out_scale on
 * tcgen05 tensor cores (shapes: proj/include/rgo/workload.hpp:44-52).
 * A and B are K-major (row-major [rows, k]); C row-major.  SwiGLU expects B
 * rows interleaved per 256-row tile as [128 gate | 128 up] and writes
 * n_out = n/2 columns.  Requirements: k*sizeof(in) % 128 == 0, 16-byte
 * aligned pointers and leading dimensions, n % 32 == 0 (n % 256 == 0 for
 * SwiGLU). */
typedef enum rgo_dtype { RGO_DT_BF16 = 0, RGO_DT_E4M3 = 1 } rgo_dtype;
typedef enum rgo_epilogue { RGO_EPI_NONE = 0, RGO_EPI_SWIGLU = 1, RGO_EPI_GELU = 2 } rgo_epilogue;

typedef struct rgo_gemm_desc {
    int32_t m, n, k;
    int32_t in_dtype;   /* rgo_dtype of A and B */
    int32_t out_dtype;  /* rgo_dtype of C */
    int32_t epilogue;   /* rgo_epilogue */
    int64_t lda, ldb, ldc; /* elements */
    float alpha;        /* dequantisation scale of A.B (sa * sb) */
    float out_scale;    /* multiplier before the output cast */
    int32_t grid;       /* 0 = one persistent CTA per SM */
    int32_t rng_warps;  /* rgo_gemm_with_rng: co-resident RNG warps per CTA, 4/6/8/12/16 (0 = 8) */
} rgo_gemm_desc;

int rgo_gemm(const rgo_gemm_desc* g, const void* d_a, const void* d_b, void* d_c,
             rgo_stream_t stream);

/* K4: the same GEMM with co-resident RNG warps (overlap mechanism B) that
 * drain the dropout-mask queue of layout m into d_bits while the tensor
 * cores run.  Whatever is left when the GEMM finishes is picked up by the
 * next rgo_gemm_with_rng on the same queue or by rgo_mask_queue_drain. */
int rgo_gemm_with_rng(const rgo_gemm_desc* g, const void* d_a, const void* d_b, void* d_c,
                      const rgo_mask_desc* m, uint8_t* d_bits, uint64_t bytes,
                      unsigned long long* d_counter, rgo_stream_t stream);

/* ------------------------------------------------------------- attention --
 * K5/K6: flash-attention forward with dropout on tcgen05 (replaces
 * attn_detail::forward_impl, proj/include/rgo/ref_attention.hpp:56-92).
 * Tensors are bf16 [batch, heads, seq, head_dim] views with element strides
 * for batch/head/position and a contiguous head dimension: the reference's
 * slice-major layout (stride_h = seq*head_dim) and the token-major QKV GEMM
 * output ([B*S, 3*H], stride_s = 3*H) are both expressible. */
typedef enum rgo_mask_source {
    RGO_MASK_NONE = 0,   /* attention_forward (ref_attention.hpp:108-110) */
    RGO_MASK_BITS = 1,   /* attention_dropout_decoupled: read d_bits (:129-146) */
    RGO_MASK_PHILOX = 2  /* attention_dropout_fused: Philox inline (:114-126) */
} rgo_mask_source;

typedef struct rgo_tensor4 {
    const void* ptr;
    int64_t stride_b, stride_h, stride_s; /* elements */
} rgo_tensor4;

typedef struct rgo_attn_desc {
    uint32_t batch, heads, seq, head_dim; /* head_dim in {64, 128} */
    float scale;          /* softmax scale; 0 = 1/sqrt(head_dim) (ref_attention.hpp:33) */
    int32_t mask_source;  /* rgo_mask_source */
    double keep_prob;     /* (0,1]; used as float like the reference (:120, :125) */
    uint64_t seed;        /* PHILOX: mask layout (batch*heads slices) seed */
    uint64_t base_offset; /* PHILOX: counter of element 0 */
    uint32_t rounds;      /* PHILOX: [1,16] */
    uint32_t flags;       /* rgo_attn_flags (0 = defaults) */
} rgo_attn_desc;

/* rgo_attn_desc.flags.  RGO_ATTN_BWD_DETERMINISTIC: head_dim-128 backward in
 * its split form -- a dK/dV kernel and a dQ kernel that accumulates dQ in
 * TMEM over all keys (no fp32 reductions across CTAs), so dQ is bitwise
 * reproducible (and equal between mask bits and inline Philox); slower than
 * the default (which reduces dQ partials with bulk fp32 adds). */
typedef enum rgo_attn_flags { RGO_ATTN_BWD_DETERMINISTIC = 1 } rgo_attn_flags;

/* O = softmax(Q K^T * scale) with dropout (denominator over all keys, kept
 * weights / keep_prob), written to o (bf16, same view convention).  d_bits
 * (MASK_BITS) is the packed mask in the reference layout for batch*heads
 * slices of seq x seq, >= ceil(B*nH*SQ^2/8) bytes.  d_lse (optional):
 * float [batch*heads*seq] natural-log row logsumexp for the backward pass. */
int rgo_attn_fwd(const rgo_attn_desc* a, const rgo_tensor4* q, const rgo_tensor4* k,
                 const rgo_tensor4* v, const uint8_t* d_bits, uint64_t bits_bytes,
                 const rgo_tensor4* o, float* d_lse, rgo_stream_t stream);

/* K7: flash-attention backward with dropout -- the training counterpart of
 * rgo_attn_fwd (the reference stops at the forward: ref_attention.hpp:56-92,
 * SPEC.md:552).  Exact derivative of the forward's semantics: with
 * P = softmax(scale Q K^T), W = keep ? P/p : 0, O = W V,
 *   dV = W^T dO,  dP = keep ? dO V^T / p : 0,  dS = P o (dP - rowsum(dO o O)),
 *   dQ = scale dS K,  dK = scale dS^T Q.
 * a, q, k, v, d_bits as for the forward (same mask source, seed, offset and
 * rounds, so the keep bits are the forward's); o and d_lse are the forward's
 * output and LSE; d_o the incoming gradient; dq/dk/dv receive bf16 gradients
 * (same view convention).  d_work: device scratch of
 * rgo_attn_bwd_workspace() bytes (fp32 dQ accumulator + per-row terms). */
int rgo_attn_bwd_workspace(const rgo_attn_desc* a, uint64_t* bytes);
int rgo_attn_bwd(const rgo_attn_desc* a, const rgo_tensor4* q, const rgo_tensor4* k,
                 const rgo_tensor4* v, const rgo_tensor4* o, const rgo_tensor4* d_o,
                 const float* d_lse, const uint8_t* d_bits, uint64_t bits_bytes,
                 const rgo_tensor4* dq, const rgo_tensor4* dk, const rgo_tensor4* dv,
                 void* d_work, uint64_t work_bytes, rgo_stream_t stream);

/* ------------------------------------------------------ host-buffer entry --
 * Drop-in forms of the reference's value-semantics API: host arrays in and
 * out, the library stages them through device memory it allocates and frees
 * inside the call (computation is on the GPU; there is no CPU path). */

/* n x philox_block on host arrays (keys n x 2, ctrs n x 4, rounds n, out n x 4). */
int rgo_philox_blocks_host(const uint32_t* h_keys, const uint32_t* h_ctrs, const int32_t* h_rounds,
                           uint32_t* h_out, uint64_t n);

/* random_attention_input (ref_attention.hpp:176-207): three float arrays of
 * slices*seq*head_dim values (q: stream 1, k: 2, v: 3). */
int rgo_random_attention_input_host(uint32_t slices, uint32_t seq, uint32_t head_dim, uint64_t seed,
                                    float* h_q, float* h_k, float* h_v);

/* attention_forward / _fused / _decoupled on reference-layout float arrays
 * (slice, pos, dim), replacing ref_attention.hpp:108-146.  head_dim <= 128:
 * the tcgen05 kernels K5/K6 (zero-padded to 64/128 on device, the softmax
 * scale stays 1/sqrt(head_dim)), inputs rounded to bf16 for the tensor cores;
 * head_dim in (128, 1024]: the fp32 CUDA-core kernel K5g on the fp32 arrays.
 * h_bits is the packed mask for RGO_MASK_BITS. */
typedef struct rgo_attn_host_desc {
    uint32_t slices, seq, head_dim;
    int32_t mask_source;  /* rgo_mask_source */
    double keep_prob;
    uint64_t seed, base_offset;
    uint32_t rounds;
    uint32_t reserved;
} rgo_attn_host_desc;

int rgo_attention_host(const rgo_attn_host_desc* a, const float* h_q, const float* h_k,
                       const float* h_v, const uint8_t* h_bits, uint64_t bits_bytes, float* h_o);

/* RNGM mask file (mask.hpp:188-297): 40-byte little-endian header
 * (magic "RNGM", u16 version 1, u16 rounds, u32 B, nH, SQ, u64 seed,
 * base_offset, f32 keep_prob) + packed payload.  Load validates magic,
 * version, rounds, truncation and padding bits (RGO_EIO on failure);
 * call with h_bits = NULL to read the header and required payload size. */
int rgo_mask_save(const char* path, const rgo_mask_desc* d, float keep_prob, const uint8_t* h_bits,
                  uint64_t bytes);
int rgo_mask_load(const char* path, rgo_mask_desc* d, float* keep_prob, uint8_t* h_bits,
                  uint64_t capacity, uint64_t* bytes);

/* FNV-1a-64 of n host bytes (offset 0xcbf29ce484222325, prime 0x100000001b3):
 * the checksum the golden mask fixtures are recorded with; lets a caller
 * self-check a device mask it copied back (bench.py's parity block). */
uint64_t rgo_fnv1a64(const uint8_t* h_data, uint64_t n);

/* ----------------------------------------------------------------- block --
 * Transformer-block step (the paper's timeline, schedule.hpp:111-136): the
 * four GEMMs between consecutive attention layers (Proj, FFN1, FFN2 of block
 * L-1 and QKV of block L, all FP8) followed by the attention of block L.
 * MoE blocks (experts > 0) replace FFN1/FFN2 by a dispatch, the per-expert
 * FFN1/FFN2 GEMMs and a combine; the RNG hides under all of them.  Routing is
 * balanced and synthetic: token-expert pair p = t*top_k + j goes to expert
 * p % experts, row p / experts of that expert's slice, gate 1/top_k.
 * Modes: SERIAL_FUSED = baseline (attention regenerates Philox inline);
 * STREAMS = mechanism A (K1 on a low-priority stream, capped grid, event join);
 * IN_GEMM = mechanism B (RNG warps co-resident in the GEMM CTAs + tail drain).
 * The caller owns every buffer; the handle owns streams, events and the
 * captured CUDA graph. */
typedef enum rgo_overlap_mode {
    RGO_OVERLAP_SERIAL_FUSED = 0,
    RGO_OVERLAP_STREAMS = 1,
    RGO_OVERLAP_IN_GEMM = 2,
    RGO_OVERLAP_NO_RNG = 3  /* measurement only: no RNG work, attention reads a stale mask */
} rgo_overlap_mode;

typedef struct rgo_block_desc {
    uint32_t batch, seq, heads, head_dim, ffn;
    int32_t gated;          /* 1: SwiGLU FFN1 with 2*ffn outputs; 0: GELU */
    double keep_prob;       /* (0,1) */
    uint32_t rounds;        /* Philox rounds */
    uint32_t use_graph;     /* capture the step into a CUDA graph */
    uint64_t seed, base_offset;  /* mask layout of batch*heads slices */
    float a_qkv, a_proj, a_ffn1, a_ffn2;  /* FP8 dequant scales */
    float s_attn, s_proj, s_ffn1, s_ffn2; /* output quantisation scales */
    rgo_launch rng_launch;  /* STREAMS: mask-kernel launch shape; IN_GEMM: rng_launch.block =
                               RNG warps per GEMM CTA (4/6/8/12/16, 0 = chosen per workload) */
    uint32_t experts;       /* 0: dense FFN; > 0: MoE with `experts` expert FFNs of width ffn */
    uint32_t top_k;         /* MoE: experts per token (balanced synthetic routing) */
    uint32_t chunks;        /* > 1: SQ-chunk pipeline (schedule.hpp:205-239, capacity.hpp:51-59):
                               the query rows of every sequence split into `chunks` windows
                               (seq/chunks % 128 == 0, dense FFN, every mode); a step is the
                               rotation [attention(c) -> Proj/FFN1/FFN2/QKV of window c] for
                               c = 0..chunks-1, reading qkv and writing qkv_out, with window c+1's
                               mask hidden under stage c's GEMMs.  The mask buffer is a 2-slot
                               ring of window masks [slice][seq/chunks][seq] (2/chunks of the full
                               mask); counter needs `chunks` entries (IN_GEMM) */
    uint32_t reserved2;
} rgo_block_desc;

typedef struct rgo_block_buffers {
    void* x;        /* e4m3 [M, d], M = batch*seq, d = heads*head_dim */
    void* wqkv;     /* e4m3 [3d, d] */
    void* wo;       /* e4m3 [d, d] */
    void* w1;       /* e4m3 [n1, d], n1 = 2*ffn (gated) or ffn */
    void* w2;       /* e4m3 [d, ffn] */
    void* qkv;      /* bf16 [M, 3d] */
    void* attn_o;   /* bf16 [M, d] */
    void* attn_o8;  /* e4m3 [M, d] */
    void* y1;       /* e4m3 [M, d] */
    void* h;        /* e4m3 [M, ffn] */
    uint8_t* mask;  /* B*nH*S^2/8 bytes */
    uint64_t mask_bytes;
    unsigned long long* counter; /* IN_GEMM work-queue counter */
    float* lse;     /* optional [B*nH*S] */
    void* xd;       /* MoE: e4m3 [M*top_k, d] dispatched expert inputs (NULL when dense) */
    void* ye;       /* MoE: bf16 [M*top_k, d] expert outputs (NULL when dense) */
    const void* attn_in; /* bf16 [M, d] step input; NULL = attn_o (steps chained through it) */
    void* qkv_out;  /* chunked step: bf16 [M, 3d] the step's QKV output (NULL when unchunked) */
} rgo_block_buffers;

typedef struct rgo_block rgo_block;

int rgo_block_create(const rgo_block_desc* d, const rgo_block_buffers* b, int32_t mode,
                     rgo_block** out);
/* Enqueue one step ordered after prior work on `stream`; *launches (optional)
 * = number of kernels the step launches. */
int rgo_block_step(rgo_block* blk, rgo_stream_t stream, int32_t* launches);
/* Device time (ms) of the last completed step: [0] GEMM window, [1] attention. */
int rgo_block_last_timings(rgo_block* blk, float* ms2);
/* Finer split: [0] GEMM window, [1] RNG tail drain / join before the attention,
 * [2] the attention kernel. */
int rgo_block_last_timings3(rgo_block* blk, float* ms3);
int rgo_block_destroy(rgo_block* blk);

/* ------------------------------------------------- tensor-parallel block --
 * Megatron TP over `size` ranks (ParallelismPlan::tp_degree,
 * capacity.hpp:14-26): heads split across ranks -- QKV and FFN1 column-
 * parallel, Proj and FFN2 row-parallel, each followed by an all-reduce done
 * by the library over peer memory (two-shot: every rank reduces M/size rows
 * of all ranks' bf16 partial sums, fused with the next GEMM's e4m3
 * quantisation, then gathers the other ranks' rows).  The rgo_block_desc
 * keeps the GLOBAL heads/ffn; buffers are the rank's: qkv [M, 3*dl],
 * attn_o/attn_in [M, dl], attn_o8 [M, dl], h [M, ffn/size], weights wqkv
 * [3*dl, d] (its heads' q, k, v rows), wo [d, dl], w1 [n1/size, d], w2
 * [d, ffn/size] (dl = heads/size*head_dim); y1 and x stay [M, d]; mask =
 * the rank's heads [rank*H/size, ...) of every batch item, compact
 * (B*H/size*S^2/8 bytes), with the global layout's keep bits and counters.
 * peer_* hold every rank's buffer as mapped in this process (rgo_ipc_open),
 * [rank] = its own.  Dense FFN, unchunked, eager (no graph). */
typedef struct rgo_block_tp {
    uint32_t size, rank;
    void* peer_part[8];  /* bf16 [M, d] partial-sum buffers */
    void* peer_y1[8];    /* e4m3 [M, d] (= each rank's buffers.y1) */
    void* peer_x[8];     /* e4m3 [M, d] (= each rank's buffers.x) */
} rgo_block_tp;

int rgo_block_create_tp(const rgo_block_desc* d, const rgo_block_buffers* b, const rgo_block_tp* tp,
                        int32_t mode, rgo_block** out);

/* One TP step: five segments, the caller's barrier(ctx) across all ranks
 * between them (called after this rank's segment has completed on the GPU). */
typedef void (*rgo_barrier_fn)(void* ctx);
int rgo_block_step_tp(rgo_block* blk, rgo_stream_t stream, rgo_barrier_fn barrier, void* ctx, int32_t* launches);

/* CUDA IPC for the peer buffers: the 64-byte handle of the device allocation
 * holding d_ptr and d_ptr's byte offset in it (caching allocators sub-allocate);
 * another process maps the allocation (rgo_ipc_open -> its base; peer access
 * enabled lazily) and adds the offset; rgo_ipc_close takes the base. */
int rgo_ipc_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset);
int rgo_ipc_open(const uint8_t* handle64, void** d_base);
int rgo_ipc_close(void* d_base);

#ifdef __cplusplus
}
#endif

#endif /* RGO_CAPI_H */
