// capi.cu -- implementation of the C-ABI boundary (include/rgo/capi.h):
// argument validation with the reference's error semantics, error mapping,
// and kernel launches.  No compute happens on the host; with no CUDA device
// every compute entry point fails with RGO_ENODEV (there is no CPU fallback).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rgo/capi.h"
#include "attn.h"
#include "block.h"
#include "gemm.h"
#include "rgo_internal.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(RGO_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

int require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(RGO_ENODEV, "no CUDA device: the rgo B200 path has no CPU fallback");
    }
    // Drop a non-sticky error that other code left in this host thread's
    // runtime state (e.g. torch's autograd worker threads), so the launch
    // checks that follow report only this call's launches.  A sticky error
    // still fails the launch itself.
    cudaGetLastError();
    return RGO_OK;
}

constexpr uint64_t kMaxBits = uint64_t{1} << 36;  // mask.hpp:108

uint64_t elem_count(const rgo_mask_desc* d) {
    return static_cast<uint64_t>(d->batch) * d->heads * d->seq * static_cast<uint64_t>(d->seq);
}

// MaskLayout::validate + rounds + threshold domain (mask.hpp:45-47, :145-146).
int validate_mask(const rgo_mask_desc* d, const char* fn) {
    if (!d) return fail(RGO_EINVAL, "%s: null descriptor", fn);
    if (elem_count(d) == 0) return fail(RGO_EINVAL, "mask layout has zero elements");
    if (d->rounds < 1 || d->rounds > 16)
        return fail(RGO_EINVAL, "%s: rounds must be in [1,16]", fn);
    if (d->threshold > (uint64_t{1} << 32))
        return fail(RGO_EINVAL, "%s: threshold must be in [0, 2^32]", fn);
    return RGO_OK;
}

}  // namespace

namespace rgo {
HostWorkspace& host_workspace() {
    static HostWorkspace ws[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return ws[dev & 63];
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}
}  // namespace rgo

extern "C" {

// internal: lets the other translation units report through rgo_last_error()
int rgo_internal_set_error(int code, const char* msg) {
    std::snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* rgo_last_error(void) { return g_err; }

int rgo_version(void) { return 1; }

int rgo_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int rgo_philox_blocks(const uint32_t* d_keys, const uint32_t* d_ctrs, const int32_t* d_rounds,
                      uint32_t* d_out, uint64_t n, rgo_stream_t stream) {
    if (int e = require_device()) return e;
    if (n && (!d_keys || !d_ctrs || !d_rounds || !d_out))
        return fail(RGO_EINVAL, "rgo_philox_blocks: null pointer");
    cudaError_t e = rgo::launch_philox_blocks(d_keys, d_ctrs, d_rounds, d_out, n,
                                              static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? RGO_OK : cuda_fail(e, "rgo_philox_blocks");
}

int rgo_keep_threshold(double p, uint64_t* threshold, float* keep_prob) {
    if (!(p >= 0.0 && p <= 1.0)) return fail(RGO_EINVAL, "keep_prob must be in [0,1]");
    const float pf = static_cast<float>(p);  // mask.hpp:59
    if (threshold)
        *threshold = static_cast<uint64_t>(std::llround(static_cast<double>(pf) * 4294967296.0));
    if (keep_prob) *keep_prob = pf;
    return RGO_OK;
}

int rgo_mask_bytes(const rgo_mask_desc* d, uint64_t* bytes) {
    if (!d) return fail(RGO_EINVAL, "rgo_mask_bytes: null descriptor");
    const uint64_t n = elem_count(d);
    if (n == 0) return fail(RGO_EINVAL, "mask layout has zero elements");
    if (bytes) *bytes = (n + 7) / 8;
    return RGO_OK;
}

int rgo_mask_generate_ex(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                         const rgo_launch* launch, rgo_stream_t stream) {
    if (int e = validate_mask(d, "rgo_mask_generate")) return e;
    if (int e = require_device()) return e;
    const uint64_t n = elem_count(d);
    if (!d_bits || bytes < (n + 7) / 8)
        return fail(RGO_EINVAL, "rgo_mask_generate: output buffer needs %llu bytes, got %llu",
                    static_cast<unsigned long long>((n + 7) / 8),
                    static_cast<unsigned long long>(bytes));
    if (reinterpret_cast<uintptr_t>(d_bits) & 15)
        return fail(RGO_EINVAL, "rgo_mask_generate: output must be 16-byte aligned");
    rgo::MaskJob j{d_bits, n, d->seed, d->base_offset, d->threshold, static_cast<int>(d->rounds)};
    rgo::LaunchShape ls;
    if (launch) {
        ls.grid = launch->grid;
        ls.block = launch->block;
        ls.dyn_smem = launch->dyn_smem;
    }
    cudaError_t e = rgo::launch_mask(j, ls, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? RGO_OK : cuda_fail(e, "rgo_mask_generate");
}

int rgo_mask_generate(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                      rgo_stream_t stream) {
    return rgo_mask_generate_ex(d, d_bits, bytes, nullptr, stream);
}

int rgo_generate_mask_host(const rgo_mask_desc* d, uint8_t* h_bits, uint64_t bytes,
                           uint32_t devices) {
    return rgo_generate_mask_host_ex(d, h_bits, bytes, devices, 0);
}

int rgo_generate_mask_host_ex(const rgo_mask_desc* d, uint8_t* h_bits, uint64_t bytes,
                              uint32_t devices, uint32_t shards) {
    if (int e = validate_mask(d, "generate_mask")) return e;
    const uint64_t n = elem_count(d);
    if (n > kMaxBits)  // mask.hpp:148-155
        return fail(RGO_EINVAL, "generate_mask: mask needs %llu bytes, guard allows %llu bytes",
                    static_cast<unsigned long long>((n + 7) / 8),
                    static_cast<unsigned long long>(kMaxBits / 8));
    const uint64_t nbytes = (n + 7) / 8;
    if (!h_bits || bytes < nbytes)
        return fail(RGO_EINVAL, "generate_mask: output buffer needs %llu bytes",
                    static_cast<unsigned long long>(nbytes));
    if (int e = require_device()) return e;
    int ndev = rgo_device_count();
    if (devices == 0 || devices > static_cast<uint32_t>(ndev)) devices = static_cast<uint32_t>(ndev);
    if (shards < devices) shards = devices;
    // Device of shard r: the caller's current device first, then the following
    // ordinals (wrapping), round-robin over `devices` -- a single-device call
    // runs on the current device, never silently on device 0.
    int prev = 0;
    cudaGetDevice(&prev);
    // Shard on 16-byte (128-element) boundaries: shard r covers elements
    // [e0, e1) and is the mask of the same layout with base_offset + e0/4,
    // so the shards concatenate to the single-device bytes (mask.hpp:139-141).
    const uint64_t nvec = (nbytes + 15) / 16;
    const uint64_t per = (nvec + shards - 1) / shards;
    std::vector<int> status(shards, RGO_OK);
    std::vector<std::string> msgs(shards);
    auto work = [&](uint32_t r) {
        const uint64_t v0 = r * per, v1 = std::min(nvec, v0 + per);
        if (v0 >= v1) return;
        const uint64_t e0 = v0 * 128, e1 = std::min(n, v1 * 128);
        const uint64_t b0 = v0 * 16, b1 = std::min(nbytes, v1 * 16);
        cudaSetDevice((prev + static_cast<int>(r % devices)) % ndev);
        // the device's staging workspace (shards sharing a device take turns on it)
        rgo::HostWorkspace& ws = rgo::host_workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        void* buf = nullptr;
        cudaError_t ce = ws.get((b1 - b0 + 15) & ~uint64_t{15}, &buf);
        if (ce != cudaSuccess) {
            status[r] = RGO_ENOMEM;
            msgs[r] = cudaGetErrorString(ce);
            return;
        }
        uint8_t* dbuf = static_cast<uint8_t*>(buf);
        rgo::MaskJob j{dbuf, e1 - e0, d->seed, d->base_offset + e0 / 4, d->threshold,
                       static_cast<int>(d->rounds)};
        ce = rgo::launch_mask(j, rgo::LaunchShape{}, nullptr);
        if (ce == cudaSuccess) ce = cudaMemcpy(h_bits + b0, dbuf, b1 - b0, cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) {
            status[r] = RGO_ECUDA;
            msgs[r] = cudaGetErrorString(ce);
        }
    };
    if (shards == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (uint32_t r = 0; r < shards; ++r) pool.emplace_back(work, r);
        for (auto& t : pool) t.join();
    }
    cudaSetDevice(prev);
    for (uint32_t r = 0; r < shards; ++r)
        if (status[r] != RGO_OK)
            return fail(status[r], "generate_mask (shard %u, device %d): %s", r,
                        (prev + static_cast<int>(r % devices)) % ndev, msgs[r].c_str());
    return RGO_OK;
}

int rgo_uniform_fill(uint64_t seed, uint32_t stream_id, uint64_t n, void* d_bf16, float* d_f32,
                     rgo_stream_t stream) {
    if (int e = require_device()) return e;
    cudaError_t e =
        rgo::launch_uniform_bf16(seed, stream_id, n, d_bf16, d_f32, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? RGO_OK : cuda_fail(e, "rgo_uniform_fill");
}

static int make_queue(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                      unsigned long long* d_counter, rgo::RngQueue* q, const char* fn) {
    if (int e = validate_mask(d, fn)) return e;
    const uint64_t n = elem_count(d);
    if (n % 128) return fail(RGO_EINVAL, "%s: queue needs B*nH*SQ^2 %% 128 == 0", fn);
    if (d->threshold == 0 || d->threshold >= (uint64_t{1} << 32))
        return fail(RGO_EINVAL, "%s: queue needs 0 < threshold < 2^32 (use rgo_mask_generate)", fn);
    if (!d_bits || bytes < n / 8 || (reinterpret_cast<uintptr_t>(d_bits) & 15))
        return fail(RGO_EINVAL, "%s: output needs %llu bytes, 16-byte aligned", fn,
                    static_cast<unsigned long long>(n / 8));
    if (!d_counter) return fail(RGO_EINVAL, "%s: null queue counter", fn);
    q->out = d_bits;
    q->n_vec = n / 128;
    q->base_offset = d->base_offset;
    q->k0 = static_cast<uint32_t>(d->seed);
    q->k1 = static_cast<uint32_t>(d->seed >> 32);
    q->thr = static_cast<uint32_t>(d->threshold);
    q->rounds = static_cast<int>(d->rounds);
    q->counter = d_counter;
    return RGO_OK;
}

int rgo_mask_queue_drain(const rgo_mask_desc* d, uint8_t* d_bits, uint64_t bytes,
                         unsigned long long* d_counter, const rgo_launch* launch,
                         rgo_stream_t stream) {
    rgo::RngQueue q{};
    if (int e = make_queue(d, d_bits, bytes, d_counter, &q, "rgo_mask_queue_drain")) return e;
    if (int e = require_device()) return e;
    cudaError_t ce = rgo::launch_rng_queue(q, launch ? launch->grid : 0, launch ? launch->block : 0,
                                           launch ? launch->dyn_smem : 0,
                                           static_cast<cudaStream_t>(stream));
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_mask_queue_drain");
}

static int gemm_job(const rgo_gemm_desc* g, const void* a, const void* b, void* c, rgo::GemmJob* j) {
    if (!g) return fail(RGO_EINVAL, "rgo_gemm: null descriptor");
    if (g->m <= 0 || g->n <= 0 || g->k <= 0) return fail(RGO_EINVAL, "rgo_gemm: dims must be >= 1");
    if (g->in_dtype != RGO_DT_BF16 && g->in_dtype != RGO_DT_E4M3)
        return fail(RGO_EINVAL, "rgo_gemm: bad input dtype");
    if (g->out_dtype != RGO_DT_BF16 && g->out_dtype != RGO_DT_E4M3)
        return fail(RGO_EINVAL, "rgo_gemm: bad output dtype");
    if (g->epilogue < RGO_EPI_NONE || g->epilogue > RGO_EPI_GELU)
        return fail(RGO_EINVAL, "rgo_gemm: bad epilogue");
    const int esz = g->in_dtype == RGO_DT_E4M3 ? 1 : 2;
    const int osz = g->out_dtype == RGO_DT_E4M3 ? 1 : 2;
    if ((static_cast<int64_t>(g->k) * esz) % 128)
        return fail(RGO_EINVAL, "rgo_gemm: k*sizeof(in) must be a multiple of 128 bytes");
    if (g->n % 32) return fail(RGO_EINVAL, "rgo_gemm: n must be a multiple of 32");
    if (g->epilogue == RGO_EPI_SWIGLU && g->n % 256)
        return fail(RGO_EINVAL, "rgo_gemm: SwiGLU needs n %% 256 == 0");
    if (g->in_dtype == RGO_DT_BF16 && g->out_dtype == RGO_DT_E4M3)
        return fail(RGO_EINVAL, "rgo_gemm: bf16 inputs produce bf16 output");
    const int n_out = g->epilogue == RGO_EPI_SWIGLU ? g->n / 2 : g->n;
    if (g->lda < g->k || g->ldb < g->k || g->ldc < n_out)
        return fail(RGO_EINVAL, "rgo_gemm: leading dimension too small");
    if (((g->lda * esz) | (g->ldb * esz) | (g->ldc * osz)) % 16)
        return fail(RGO_EINVAL, "rgo_gemm: leading dimensions must be 16-byte multiples");
    if (!a || !b || !c || ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                            reinterpret_cast<uintptr_t>(c)) & 15))
        return fail(RGO_EINVAL, "rgo_gemm: pointers must be non-null and 16-byte aligned");
    j->fp8 = g->in_dtype == RGO_DT_E4M3;
    j->M = g->m; j->N = g->n; j->K = g->k;
    j->A = a; j->lda = g->lda; j->B = b; j->ldb = g->ldb; j->C = c; j->ldc = g->ldc;
    j->epi = g->epilogue;
    j->out = g->out_dtype == RGO_DT_E4M3 ? rgo_gk::OUT_E4M3 : rgo_gk::OUT_BF16;
    j->alpha = g->alpha; j->out_scale = g->out_scale; j->grid = g->grid; j->rng = nullptr;
    const int rw = g->rng_warps;
    if (rw != 0 && rw != 4 && rw != 6 && rw != 8 && rw != 12 && rw != 16)
        return fail(RGO_EINVAL, "gemm: rng_warps must be 0, 4, 6, 8, 12 or 16 (got %d)", rw);
    j->rng_warps = rw;
    return RGO_OK;
}

int rgo_gemm(const rgo_gemm_desc* g, const void* d_a, const void* d_b, void* d_c,
             rgo_stream_t stream) {
    rgo::GemmJob j{};
    if (int e = gemm_job(g, d_a, d_b, d_c, &j)) return e;
    if (int e = require_device()) return e;
    cudaError_t ce = rgo::launch_gemm(j, static_cast<cudaStream_t>(stream));
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_gemm");
}

int rgo_gemm_with_rng(const rgo_gemm_desc* g, const void* d_a, const void* d_b, void* d_c,
                      const rgo_mask_desc* m, uint8_t* d_bits, uint64_t bytes,
                      unsigned long long* d_counter, rgo_stream_t stream) {
    rgo::GemmJob j{};
    if (int e = gemm_job(g, d_a, d_b, d_c, &j)) return e;
    rgo::RngQueue q{};
    if (int e = make_queue(m, d_bits, bytes, d_counter, &q, "rgo_gemm_with_rng")) return e;
    if (int e = require_device()) return e;
    j.rng = &q;
    cudaError_t ce = rgo::launch_gemm(j, static_cast<cudaStream_t>(stream));
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_gemm_with_rng");
}

// Validation shared by the forward and backward (ref_attention.hpp:117-118,
// :131-139 for the dropout arguments).
static int attn_check(const char* fn, const rgo_attn_desc* a, const uint8_t* d_bits, uint64_t bits_bytes) {
    if (a->batch < 1 || a->heads < 1 || a->seq < 1 || a->head_dim < 1)
        return fail(RGO_EINVAL, "attention dims must be >= 1");
    if (a->head_dim != 64 && a->head_dim != 128)
        return fail(RGO_EINVAL, "%s: head_dim must be 64 or 128 (pad smaller heads)", fn);
    if (a->mask_source < RGO_MASK_NONE || a->mask_source > RGO_MASK_PHILOX)
        return fail(RGO_EINVAL, "%s: bad mask source", fn);
    const bool drop = a->mask_source != RGO_MASK_NONE;
    if (drop && !(a->keep_prob > 0.0 && a->keep_prob <= 1.0))  // ref_attention.hpp:117-118
        return fail(RGO_EINVAL, "attention_dropout: p must be in (0,1]");
    const uint64_t n = static_cast<uint64_t>(a->batch) * a->heads * a->seq * static_cast<uint64_t>(a->seq);
    if (a->mask_source == RGO_MASK_BITS && (!d_bits || bits_bytes < (n + 7) / 8))
        return fail(RGO_EINVAL, "attention_dropout_decoupled: mask needs %llu bytes",
                    static_cast<unsigned long long>((n + 7) / 8));
    if (a->mask_source == RGO_MASK_PHILOX && (a->rounds < 1 || a->rounds > 16))
        return fail(RGO_EINVAL, "attention_dropout_fused: rounds must be in [1,16]");
    return RGO_OK;
}

static int tensors_ok(const char* fn, const rgo_tensor4* const* ts, int n) {
    for (int i = 0; i < n; ++i) {
        const rgo_tensor4* t = ts[i];
        if (!t || !t->ptr || (reinterpret_cast<uintptr_t>(t->ptr) & 15) ||
            ((t->stride_b | t->stride_h | t->stride_s) * 2) % 16)
            return fail(RGO_EINVAL, "%s: tensors need 16-byte aligned base and strides", fn);
    }
    return RGO_OK;
}

extern "C++" {
// The dropout fields shared by AttnJob and AttnBwdJob.
template <class J>
static void attn_fill(J& j, const rgo_attn_desc* a, const uint8_t* d_bits, uint64_t bits_bytes) {
    j.B = static_cast<int>(a->batch);
    j.H = static_cast<int>(a->heads);
    j.S = static_cast<int>(a->seq);
    j.HD = static_cast<int>(a->head_dim);
    j.scale = a->scale > 0 ? a->scale : 1.0f / std::sqrt(static_cast<float>(a->head_dim));
    j.mode = a->mask_source;
    float kp = 1.0f;
    uint64_t thr = uint64_t{1} << 32;
    rgo_keep_threshold(a->mask_source != RGO_MASK_NONE ? a->keep_prob : 1.0, &thr, &kp);
    j.keep_prob = kp;
    j.threshold = thr;
    j.bits = d_bits;
    j.bits_bytes = bits_bytes;
    j.seed = a->seed;
    j.base_offset = a->base_offset;
    j.rounds = static_cast<int>(a->rounds);
}

static rgo::AttnTensor view(const rgo_tensor4* t) { return {t->ptr, t->stride_b, t->stride_h, t->stride_s}; }
static rgo::AttnOut view_out(const rgo_tensor4* t) {
    return {const_cast<void*>(t->ptr), t->stride_b, t->stride_h, t->stride_s};
}
}  // extern "C++"

int rgo_attn_fwd(const rgo_attn_desc* a, const rgo_tensor4* q, const rgo_tensor4* k,
                 const rgo_tensor4* v, const uint8_t* d_bits, uint64_t bits_bytes,
                 const rgo_tensor4* o, float* d_lse, rgo_stream_t stream) {
    if (!a || !q || !k || !v || !o) return fail(RGO_EINVAL, "rgo_attn_fwd: null argument");
    if (int e = attn_check("rgo_attn_fwd", a, d_bits, bits_bytes)) return e;
    const rgo_tensor4* ts[4] = {q, k, v, o};
    if (int e = tensors_ok("rgo_attn_fwd", ts, 4)) return e;
    if (int e = require_device()) return e;
    rgo::AttnJob j{};
    attn_fill(j, a, d_bits, bits_bytes);
    j.q = view(q);
    j.k = view(k);
    j.v = view(v);
    j.o = view_out(o);
    j.lse = d_lse;
    cudaError_t ce = rgo::launch_attn_fwd(j, static_cast<cudaStream_t>(stream));
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_attn_fwd");
}

int rgo_attn_bwd_workspace(const rgo_attn_desc* a, uint64_t* bytes) {
    if (!a || !bytes) return fail(RGO_EINVAL, "rgo_attn_bwd_workspace: null argument");
    if (a->batch < 1 || a->heads < 1 || a->seq < 1 || (a->head_dim != 64 && a->head_dim != 128))
        return fail(RGO_EINVAL, "rgo_attn_bwd_workspace: bad dims (head_dim must be 64 or 128)");
    *bytes = rgo::attn_bwd_workspace_bytes(static_cast<int>(a->batch), static_cast<int>(a->heads),
                                           static_cast<int>(a->seq), static_cast<int>(a->head_dim));
    return RGO_OK;
}

int rgo_attn_bwd(const rgo_attn_desc* a, const rgo_tensor4* q, const rgo_tensor4* k, const rgo_tensor4* v,
                 const rgo_tensor4* o, const rgo_tensor4* d_o, const float* d_lse, const uint8_t* d_bits,
                 uint64_t bits_bytes, const rgo_tensor4* dq, const rgo_tensor4* dk, const rgo_tensor4* dv,
                 void* d_work, uint64_t work_bytes, rgo_stream_t stream) {
    if (!a || !q || !k || !v || !o || !d_o || !dq || !dk || !dv || !d_lse)
        return fail(RGO_EINVAL, "rgo_attn_bwd: null argument");
    if (int e = attn_check("rgo_attn_bwd", a, d_bits, bits_bytes)) return e;
    const rgo_tensor4* ts[8] = {q, k, v, o, d_o, dq, dk, dv};
    if (int e = tensors_ok("rgo_attn_bwd", ts, 8)) return e;
    const uint64_t need = rgo::attn_bwd_workspace_bytes(static_cast<int>(a->batch), static_cast<int>(a->heads),
                                                        static_cast<int>(a->seq), static_cast<int>(a->head_dim));
    if (!d_work || work_bytes < need || (reinterpret_cast<uintptr_t>(d_work) & 15))
        return fail(RGO_EINVAL, "rgo_attn_bwd: workspace needs %llu bytes (16-byte aligned)",
                    static_cast<unsigned long long>(need));
    if (int e = require_device()) return e;
    rgo::AttnBwdJob j{};
    attn_fill(j, a, d_bits, bits_bytes);
    j.q = view(q);
    j.k = view(k);
    j.v = view(v);
    j.o = view(o);
    j.dout = view(d_o);
    j.dq = view_out(dq);
    j.dk = view_out(dk);
    j.dv = view_out(dv);
    j.lse = d_lse;
    j.work = d_work;
    j.deterministic = (a->flags & RGO_ATTN_BWD_DETERMINISTIC) != 0;
    cudaError_t ce = rgo::launch_attn_bwd(j, static_cast<cudaStream_t>(stream));
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_attn_bwd");
}

struct rgo_block {
    rgo::Block* impl;
};

int rgo_block_create(const rgo_block_desc* d, const rgo_block_buffers* b, int32_t mode, rgo_block** out) {
    if (!d || !b || !out) return fail(RGO_EINVAL, "rgo_block_create: null argument");
    if (mode < RGO_OVERLAP_SERIAL_FUSED || mode > RGO_OVERLAP_NO_RNG)
        return fail(RGO_EINVAL, "rgo_block_create: bad overlap mode");
    if (d->head_dim != 64 && d->head_dim != 128) return fail(RGO_EINVAL, "rgo_block_create: head_dim 64/128");
    if (!(d->keep_prob > 0.0 && d->keep_prob < 1.0)) return fail(RGO_EINVAL, "rgo_block_create: keep_prob in (0,1)");
    if (d->rounds < 1 || d->rounds > 16) return fail(RGO_EINVAL, "rgo_block_create: rounds must be in [1,16]");
    {
        // keep_prob is used as a float (mask.hpp:59): a double in (0,1) can still round
        // to a threshold of 0 (keep nothing) or 2^32 (keep all), which the in-GEMM
        // queue's 32-bit compare cannot express -- the modes would silently disagree
        uint64_t thr0 = 0;
        rgo_keep_threshold(d->keep_prob, &thr0, nullptr);
        if (thr0 == 0 || thr0 >= (uint64_t{1} << 32))
            return fail(RGO_EINVAL, "rgo_block_create: keep_prob %.17g rounds (as float) to a threshold of %llu; "
                                    "needs 0 < threshold < 2^32", d->keep_prob, static_cast<unsigned long long>(thr0));
    }
    if (mode == RGO_OVERLAP_IN_GEMM) {
        const uint32_t rw = d->rng_launch.block;
        if (rw != 0 && rw != 4 && rw != 6 && rw != 8 && rw != 12 && rw != 16)
            return fail(RGO_EINVAL, "rgo_block_create: IN_GEMM rng_launch.block = RNG warps per GEMM CTA must be "
                                    "0, 4, 6, 8, 12 or 16 (got %u)", rw);
    }
    const uint64_t dm = static_cast<uint64_t>(d->heads) * d->head_dim;
    if (dm % 256 || d->ffn % 128 || (static_cast<uint64_t>(d->batch) * d->seq) % 128 || d->seq % 128)
        return fail(RGO_EINVAL, "rgo_block_create: needs d %% 256, ffn %% 128, seq %% 128 == 0");
    if (d->gated && d->ffn % 128) return fail(RGO_EINVAL, "rgo_block_create: gated ffn %% 128");
    if (d->experts) {
        const uint64_t pairs = static_cast<uint64_t>(d->batch) * d->seq * d->top_k;
        if (d->top_k < 1 || d->top_k > d->experts || pairs % d->experts || (pairs / d->experts) % 128)
            return fail(RGO_EINVAL, "rgo_block_create: MoE needs 1 <= top_k <= experts and "
                                    "(batch*seq*top_k/experts) %% 128 == 0");
        if (!b->xd || !b->ye) return fail(RGO_EINVAL, "rgo_block_create: MoE needs the xd and ye buffers");
    }
    const uint32_t chunks = d->chunks > 1 ? d->chunks : 1;
    if (chunks > 1 && (d->seq % chunks || (d->seq / chunks) % 128 || d->experts))
        return fail(RGO_EINVAL, "pipeline_schedule: chunks must divide SQ (into windows of a multiple of 128 rows; "
                                "dense FFN)");
    if (chunks > 64) return fail(RGO_EINVAL, "rgo_block_create: at most 64 chunks");
    if (chunks > 1 && !b->qkv_out) return fail(RGO_EINVAL, "rgo_block_create: chunked step needs qkv_out");
    const uint64_t n_full = static_cast<uint64_t>(d->batch) * d->heads * d->seq * static_cast<uint64_t>(d->seq);
    const uint64_t n = chunks > 1 ? 2 * (n_full / chunks) : n_full;  // chunked: 2-slot ring of window masks
    if (!b->mask || b->mask_bytes < n / 8 || !b->counter || !b->x || !b->wqkv || !b->wo || !b->w1 || !b->w2 ||
        !b->qkv || !b->attn_o || !b->attn_o8 || !b->y1 || !b->h)
        return fail(RGO_EINVAL, "rgo_block_create: missing buffer (mask needs %llu bytes)",
                    static_cast<unsigned long long>(n / 8));
    if (int e = require_device()) return e;
    rgo::BlockConfig c{};
    c.batch = static_cast<int>(d->batch); c.seq = static_cast<int>(d->seq);
    c.heads = static_cast<int>(d->heads); c.head_dim = static_cast<int>(d->head_dim);
    c.ffn = static_cast<int>(d->ffn); c.gated = d->gated;
    uint64_t thr = 0;
    float kp = 0;
    rgo_keep_threshold(d->keep_prob, &thr, &kp);
    c.keep_prob = kp; c.threshold = thr; c.rounds = static_cast<int>(d->rounds);
    c.seed = d->seed; c.base_offset = d->base_offset;
    c.a_qkv = d->a_qkv; c.a_proj = d->a_proj; c.a_ffn1 = d->a_ffn1; c.a_ffn2 = d->a_ffn2;
    c.s_attn = d->s_attn; c.s_proj = d->s_proj; c.s_ffn1 = d->s_ffn1; c.s_ffn2 = d->s_ffn2;
    c.rng_grid = d->rng_launch.grid; c.rng_block = d->rng_launch.block; c.rng_smem = d->rng_launch.dyn_smem;
    c.experts = static_cast<int>(d->experts);
    c.top_k = static_cast<int>(d->top_k);
    c.chunks = static_cast<int>(chunks);
    rgo::BlockBuffers bb{b->x, b->wqkv, b->wo, b->w1, b->w2, b->qkv, b->attn_o, b->attn_o8, b->y1, b->h,
                         b->mask, b->mask_bytes, b->counter, b->lse, b->xd, b->ye, b->attn_in, b->qkv_out};
    rgo::Block* impl = nullptr;
    cudaError_t ce = rgo::block_create(c, bb, mode, d->use_graph != 0, &impl);
    if (ce != cudaSuccess) return cuda_fail(ce, "rgo_block_create");
    *out = new rgo_block{impl};
    return RGO_OK;
}

int rgo_block_create_tp(const rgo_block_desc* d, const rgo_block_buffers* b, const rgo_block_tp* tp, int32_t mode,
                        rgo_block** out) {
    if (!d || !b || !tp || !out) return fail(RGO_EINVAL, "rgo_block_create_tp: null argument");
    const uint32_t n = tp->size, r = tp->rank;
    if (n < 2 || n > 8 || r >= n) return fail(RGO_EINVAL, "rgo_block_create_tp: size in [2, 8], rank < size");
    if (d->heads % n) return fail(RGO_EINVAL, "tp_degree must divide nH");  // capacity.hpp:22-23
    if (d->experts || d->chunks > 1) return fail(RGO_EINVAL, "rgo_block_create_tp: dense FFN, unchunked step");
    const uint64_t dl = static_cast<uint64_t>(d->heads / n) * d->head_dim, M = static_cast<uint64_t>(d->batch) * d->seq;
    if (dl % 128 || (d->ffn / n) % 128 || d->ffn % n || M % (128 * n))
        return fail(RGO_EINVAL, "rgo_block_create_tp: needs (heads/size)*head_dim %% 128, (ffn/size) %% 128 and "
                                "batch*seq %% (128*size) == 0");
    for (uint32_t t = 0; t < n; ++t)
        if (!tp->peer_part[t] || !tp->peer_y1[t] || !tp->peer_x[t])
            return fail(RGO_EINVAL, "rgo_block_create_tp: missing peer buffer of rank %u", t);
    if (tp->peer_y1[r] != b->y1 || tp->peer_x[r] != b->x)
        return fail(RGO_EINVAL, "rgo_block_create_tp: peer_y1/peer_x[rank] must be this rank's y1/x");
    {  // the rank's compact mask: B * (H/size) * S^2 bits
        const uint64_t need = static_cast<uint64_t>(d->batch) * (d->heads / n) * d->seq * static_cast<uint64_t>(d->seq) / 8;
        if (!b->mask || b->mask_bytes < need || !b->counter || !b->x || !b->wqkv || !b->wo || !b->w1 || !b->w2 ||
            !b->qkv || !b->attn_o || !b->attn_o8 || !b->y1 || !b->h)
            return fail(RGO_EINVAL, "rgo_block_create_tp: missing buffer (mask needs %llu bytes)",
                        static_cast<unsigned long long>(need));
    }
    if (mode < RGO_OVERLAP_SERIAL_FUSED || mode > RGO_OVERLAP_NO_RNG)
        return fail(RGO_EINVAL, "rgo_block_create_tp: bad overlap mode");
    if (d->head_dim != 64 && d->head_dim != 128) return fail(RGO_EINVAL, "rgo_block_create_tp: head_dim 64/128");
    if (d->rounds < 1 || d->rounds > 16) return fail(RGO_EINVAL, "rgo_block_create_tp: rounds must be in [1,16]");
    uint64_t thr = 0;
    float kp = 0;
    if (rgo_keep_threshold(d->keep_prob, &thr, &kp) != RGO_OK || thr == 0 || thr >= (uint64_t{1} << 32))
        return fail(RGO_EINVAL, "rgo_block_create_tp: keep_prob must give 0 < threshold < 2^32");
    if (mode == RGO_OVERLAP_IN_GEMM) {
        const uint32_t rw = d->rng_launch.block;
        if (rw != 0 && rw != 4 && rw != 6 && rw != 8 && rw != 12 && rw != 16)
            return fail(RGO_EINVAL, "rgo_block_create_tp: IN_GEMM RNG warps per GEMM CTA must be 0/4/6/8/12/16");
    }
    if (int e = require_device()) return e;
    rgo::BlockConfig c{};
    c.batch = static_cast<int>(d->batch); c.seq = static_cast<int>(d->seq);
    c.heads = static_cast<int>(d->heads); c.head_dim = static_cast<int>(d->head_dim);
    c.ffn = static_cast<int>(d->ffn); c.gated = d->gated;
    c.keep_prob = kp; c.threshold = thr; c.rounds = static_cast<int>(d->rounds);
    c.seed = d->seed; c.base_offset = d->base_offset;
    c.a_qkv = d->a_qkv; c.a_proj = d->a_proj; c.a_ffn1 = d->a_ffn1; c.a_ffn2 = d->a_ffn2;
    c.s_attn = d->s_attn; c.s_proj = d->s_proj; c.s_ffn1 = d->s_ffn1; c.s_ffn2 = d->s_ffn2;
    c.rng_grid = d->rng_launch.grid; c.rng_block = d->rng_launch.block; c.rng_smem = d->rng_launch.dyn_smem;
    c.experts = 0; c.top_k = 0; c.chunks = 1;
    c.tp_size = static_cast<int>(n); c.tp_rank = static_cast<int>(r);
    rgo::BlockBuffers bb{b->x, b->wqkv, b->wo, b->w1, b->w2, b->qkv, b->attn_o, b->attn_o8, b->y1, b->h,
                         b->mask, b->mask_bytes, b->counter, b->lse, nullptr, nullptr, b->attn_in, nullptr};
    for (uint32_t t = 0; t < n; ++t) {
        bb.peer_part[t] = tp->peer_part[t];
        bb.peer_y1[t] = tp->peer_y1[t];
        bb.peer_x[t] = tp->peer_x[t];
    }
    rgo::Block* impl = nullptr;
    cudaError_t ce = rgo::block_create(c, bb, mode, false, &impl);
    if (ce != cudaSuccess) return cuda_fail(ce, "rgo_block_create_tp");
    *out = new rgo_block{impl};
    return RGO_OK;
}

int rgo_block_step_tp(rgo_block* blk, rgo_stream_t stream, rgo_barrier_fn barrier, void* ctx, int32_t* launches) {
    if (!blk || !barrier) return fail(RGO_EINVAL, "rgo_block_step_tp: null argument");
    if (rgo::block_tp_size(blk->impl) < 2)
        return fail(RGO_EINVAL, "rgo_block_step_tp: not a tensor-parallel block (use rgo_block_step)");
    int n = 0;
    cudaError_t ce = rgo::block_step_tp(blk->impl, static_cast<cudaStream_t>(stream), barrier, ctx, &n);
    if (launches) *launches = n;
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_block_step_tp");
}

// Base of the device allocation holding d_ptr (caching allocators sub-allocate: an
// IPC handle names the whole allocation, so the offset has to travel with it).
static cudaError_t alloc_base(const void* d_ptr, uintptr_t* base) {
    using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
                       q == cudaDriverEntryPointSuccess
                   ? reinterpret_cast<Fn>(p)
                   : nullptr;
    }();
    if (!fn) return cudaErrorNotSupported;
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) return cudaErrorInvalidValue;
    *base = static_cast<uintptr_t>(b);
    return cudaSuccess;
}

int rgo_ipc_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset) {
    if (!d_ptr || !handle64 || !offset) return fail(RGO_EINVAL, "rgo_ipc_handle: null argument");
    if (int e = require_device()) return e;
    uintptr_t base = 0;
    cudaError_t ce = alloc_base(d_ptr, &base);
    if (ce != cudaSuccess) return cuda_fail(ce, "rgo_ipc_handle: allocation base");
    cudaIpcMemHandle_t h;
    ce = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
    if (ce != cudaSuccess) return cuda_fail(ce, "rgo_ipc_handle");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, 64);
    *offset = static_cast<uint64_t>(reinterpret_cast<uintptr_t>(d_ptr) - base);
    return RGO_OK;
}

int rgo_ipc_open(const uint8_t* handle64, void** d_base) {
    if (!handle64 || !d_base) return fail(RGO_EINVAL, "rgo_ipc_open: null argument");
    if (int e = require_device()) return e;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    cudaError_t ce = cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess);
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_ipc_open");
}

int rgo_ipc_close(void* d_base) {
    if (!d_base) return fail(RGO_EINVAL, "rgo_ipc_close: null argument");
    cudaError_t ce = cudaIpcCloseMemHandle(d_base);
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_ipc_close");
}

int rgo_block_step(rgo_block* blk, rgo_stream_t stream, int32_t* launches) {
    if (!blk) return fail(RGO_EINVAL, "rgo_block_step: null handle");
    if (rgo::block_tp_size(blk->impl) > 1)
        return fail(RGO_EINVAL, "rgo_block_step: a tensor-parallel block steps with rgo_block_step_tp");
    int n = 0;
    cudaError_t ce = rgo::block_step(blk->impl, static_cast<cudaStream_t>(stream), &n);
    if (launches) *launches = n;
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_block_step");
}

int rgo_block_last_timings(rgo_block* blk, float* ms2) {
    if (!blk || !ms2) return fail(RGO_EINVAL, "rgo_block_last_timings: null argument");
    cudaError_t ce = rgo::block_last_timings(blk->impl, ms2);
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_block_last_timings");
}

int rgo_block_last_timings3(rgo_block* blk, float* ms3) {
    if (!blk || !ms3) return fail(RGO_EINVAL, "rgo_block_last_timings3: null argument");
    cudaError_t ce = rgo::block_last_timings3(blk->impl, ms3);
    return ce == cudaSuccess ? RGO_OK : cuda_fail(ce, "rgo_block_last_timings3");
}

int rgo_block_destroy(rgo_block* blk) {
    if (!blk) return RGO_OK;
    rgo::block_destroy(blk->impl);
    delete blk;
    return RGO_OK;
}

}  // extern "C"
