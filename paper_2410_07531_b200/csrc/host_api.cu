// host_api.cu -- host-buffer entry points of the C ABI (include/rgo/capi.h):
// the value-semantics forms the reference's C++ API needs (philox_block,
// random_attention_input, attention_*, RNGM mask files).  Device staging comes
// from a per-device grow-only workspace (rgo::host_workspace) or, for the rare
// philox/random-input helpers, is allocated inside the call; all arithmetic
// runs on the GPU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>

#include "attn.h"
#include "rgo/capi.h"
#include "rgo_internal.h"

namespace {

thread_local char g_msg[512];

// Shares rgo_last_error()'s buffer through the exported setter below.
int set_error(int code, const char* fmt, ...);

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, n ? n : 1); }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// fp32 [slices, seq, hd] (host layout of ref_attention.hpp:20-31) -> bf16
// [slices, seq, hp] zero-padded in the head dimension.
__global__ void pad_to_bf16(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, uint64_t rows, int hd,
                            int hp) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * hp) return;
    const uint64_t r = i / hp;
    const int d = static_cast<int>(i % hp);
    out[i] = __float2bfloat16_rn(d < hd ? in[r * hd + d] : 0.0f);
}

__global__ void unpad_to_f32(const __nv_bfloat16* __restrict__ in, float* __restrict__ out, uint64_t rows, int hd,
                             int hp) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * hd) return;
    const uint64_t r = i / hd;
    const int d = static_cast<int>(i % hd);
    out[i] = __bfloat162float(in[r * hp + d]);
}

unsigned blocks_for(uint64_t n) { return static_cast<unsigned>((n + 255) / 256); }

// little-endian field packing for the RNGM header (mask.hpp:188-201)
void put(uint8_t* p, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
uint64_t get(const uint8_t* p, int bytes) {
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

}  // namespace

extern "C" int rgo_internal_set_error(int code, const char* msg);

namespace {
int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    return rgo_internal_set_error(code, g_msg);
}
int cuda_error(cudaError_t e, const char* where) {
    return set_error(RGO_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}
}  // namespace

#define RGO_TRY(expr, where)                         \
    do {                                             \
        cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) return cuda_error(e_, where); \
    } while (0)

extern "C" {

int rgo_philox_blocks_host(const uint32_t* h_keys, const uint32_t* h_ctrs, const int32_t* h_rounds,
                           uint32_t* h_out, uint64_t n) {
    if (n == 0) return RGO_OK;
    if (!h_keys || !h_ctrs || !h_rounds || !h_out) return set_error(RGO_EINVAL, "philox_block: null pointer");
    for (uint64_t i = 0; i < n; ++i)
        if (h_rounds[i] < 1 || h_rounds[i] > 16)  // philox.hpp:86-87
            return set_error(RGO_EINVAL, "philox_block: rounds must be in [1,16]");
    if (rgo_device_count() == 0) return set_error(RGO_ENODEV, "no CUDA device: the rgo B200 path has no CPU fallback");
    DevBuf k, c, r, o;
    RGO_TRY(k.alloc(n * 8), "philox_block");
    RGO_TRY(c.alloc(n * 16), "philox_block");
    RGO_TRY(r.alloc(n * 4), "philox_block");
    RGO_TRY(o.alloc(n * 16), "philox_block");
    RGO_TRY(cudaMemcpy(k.p, h_keys, n * 8, cudaMemcpyHostToDevice), "philox_block");
    RGO_TRY(cudaMemcpy(c.p, h_ctrs, n * 16, cudaMemcpyHostToDevice), "philox_block");
    RGO_TRY(cudaMemcpy(r.p, h_rounds, n * 4, cudaMemcpyHostToDevice), "philox_block");
    int rc = rgo_philox_blocks(k.as<uint32_t>(), c.as<uint32_t>(), r.as<int32_t>(), o.as<uint32_t>(), n, nullptr);
    if (rc != RGO_OK) return rc;
    RGO_TRY(cudaMemcpy(h_out, o.p, n * 16, cudaMemcpyDeviceToHost), "philox_block");
    return RGO_OK;
}

int rgo_random_attention_input_host(uint32_t slices, uint32_t seq, uint32_t head_dim, uint64_t seed,
                                    float* h_q, float* h_k, float* h_v) {
    const uint64_t n = static_cast<uint64_t>(slices) * seq * head_dim;
    if (n == 0) return set_error(RGO_EINVAL, "attention dims must be >= 1");
    if (rgo_device_count() == 0) return set_error(RGO_ENODEV, "no CUDA device: the rgo B200 path has no CPU fallback");
    DevBuf d;
    RGO_TRY(d.alloc(n * 4), "random_attention_input");
    float* outs[3] = {h_q, h_k, h_v};
    for (uint32_t s = 0; s < 3; ++s) {
        int rc = rgo_uniform_fill(seed, s + 1, n, nullptr, d.as<float>(), nullptr);
        if (rc != RGO_OK) return rc;
        RGO_TRY(cudaMemcpy(outs[s], d.p, n * 4, cudaMemcpyDeviceToHost), "random_attention_input");
    }
    return RGO_OK;
}

// head_dim > 128: the fp32 CUDA-core kernel (K5g) on the reference's own fp32 arrays.
static int attention_host_generic(const rgo_attn_host_desc* a, const float* h_q, const float* h_k, const float* h_v,
                                  const uint8_t* h_bits, uint64_t bits_bytes, float* h_o) {
    const uint64_t n = static_cast<uint64_t>(a->slices) * a->seq * a->head_dim;
    auto up = [](uint64_t x) { return (x + 255) & ~uint64_t{255}; };
    const uint64_t f_bytes = up(n * 4), b_bytes = a->mask_source == RGO_MASK_BITS ? up(bits_bytes) : 0;
    rgo::HostWorkspace& ws = rgo::host_workspace();
    std::lock_guard<std::mutex> lk(ws.mu);
    void* base = nullptr;
    RGO_TRY(ws.get(4 * f_bytes + b_bytes, &base), "attention");
    uint8_t* w8 = static_cast<uint8_t*>(base);
    float* d[4];
    for (int t = 0; t < 4; ++t) d[t] = reinterpret_cast<float*>(w8 + t * f_bytes);
    const float* hs[3] = {h_q, h_k, h_v};
    for (int t = 0; t < 3; ++t) RGO_TRY(cudaMemcpy(d[t], hs[t], n * 4, cudaMemcpyHostToDevice), "attention");
    const uint8_t* dbits = nullptr;
    if (a->mask_source == RGO_MASK_BITS) {
        uint8_t* bits = w8 + 4 * f_bytes;
        RGO_TRY(cudaMemcpy(bits, h_bits, bits_bytes, cudaMemcpyHostToDevice), "attention");
        dbits = bits;
    }
    uint64_t thr = 0;
    float kp = 1.0f;  // the float keep probability the reference scales by (ref_attention.hpp:120,125)
    if (a->mask_source != RGO_MASK_NONE) {
        int rc = rgo_keep_threshold(a->keep_prob, &thr, &kp);
        if (rc != RGO_OK) return rc;
    }
    const float scale = 1.0f / std::sqrt(static_cast<float>(a->head_dim));  // ref_attention.hpp:33
    RGO_TRY(rgo::launch_attn_generic_f32(d[0], d[1], d[2], d[3], a->slices, a->seq, a->head_dim, scale,
                                         a->mask_source, kp, dbits, a->seed, thr, a->base_offset,
                                         a->rounds, nullptr),
            "attention");
    RGO_TRY(cudaMemcpy(h_o, d[3], n * 4, cudaMemcpyDeviceToHost), "attention");
    return RGO_OK;
}

int rgo_attention_host(const rgo_attn_host_desc* a, const float* h_q, const float* h_k, const float* h_v,
                       const uint8_t* h_bits, uint64_t bits_bytes, float* h_o) {
    if (!a || !h_q || !h_k || !h_v || !h_o) return set_error(RGO_EINVAL, "attention: null argument");
    if (a->slices < 1 || a->seq < 1 || a->head_dim < 1) return set_error(RGO_EINVAL, "attention dims must be >= 1");
    if (a->head_dim > rgo::kGenericMaxHeadDim) return set_error(RGO_EINVAL, "attention: head_dim > 1024 not supported");
    if (rgo_device_count() == 0) return set_error(RGO_ENODEV, "no CUDA device: the rgo B200 path has no CPU fallback");
    const int hd = static_cast<int>(a->head_dim), hp = hd <= 64 ? 64 : 128;
    const uint64_t rows = static_cast<uint64_t>(a->slices) * a->seq;
    if (a->mask_source == RGO_MASK_BITS && !h_bits)
        return set_error(RGO_EINVAL, "attention_dropout_decoupled: null mask");
    if (hd > 128) return attention_host_generic(a, h_q, h_k, h_v, h_bits, bits_bytes, h_o);
    // one staging allocation per device, reused across calls: f32 rows, q, k, v, o (bf16), bits
    auto up = [](uint64_t n) { return (n + 255) & ~uint64_t{255}; };
    const uint64_t f_bytes = up(rows * hd * 4), t_bytes = up(rows * hp * 2),
                   b_bytes = a->mask_source == RGO_MASK_BITS ? up(bits_bytes) : 0;
    rgo::HostWorkspace& ws = rgo::host_workspace();
    std::lock_guard<std::mutex> lk(ws.mu);
    void* base = nullptr;
    RGO_TRY(ws.get(f_bytes + 4 * t_bytes + b_bytes, &base), "attention");
    uint8_t* w8 = static_cast<uint8_t*>(base);
    float* f = reinterpret_cast<float*>(w8);
    __nv_bfloat16* ds[4];
    for (int t = 0; t < 4; ++t) ds[t] = reinterpret_cast<__nv_bfloat16*>(w8 + f_bytes + t * t_bytes);
    const float* hs[3] = {h_q, h_k, h_v};
    for (int t = 0; t < 3; ++t) {
        RGO_TRY(cudaMemcpy(f, hs[t], rows * hd * 4, cudaMemcpyHostToDevice), "attention");
        pad_to_bf16<<<blocks_for(rows * hp), 256>>>(f, ds[t], rows, hd, hp);
        RGO_TRY(cudaGetLastError(), "attention");
    }
    const uint8_t* dbits = nullptr;
    if (a->mask_source == RGO_MASK_BITS) {
        uint8_t* bits = w8 + f_bytes + 4 * t_bytes;
        RGO_TRY(cudaMemcpy(bits, h_bits, bits_bytes, cudaMemcpyHostToDevice), "attention");
        dbits = bits;
    }
    rgo_attn_desc d{};
    d.batch = 1;
    d.heads = a->slices;
    d.seq = a->seq;
    d.head_dim = static_cast<uint32_t>(hp);
    d.scale = 1.0f / std::sqrt(static_cast<float>(hd));  // ref_attention.hpp:33 with the true head_dim
    d.mask_source = a->mask_source;
    d.keep_prob = a->keep_prob;
    d.seed = a->seed;
    d.base_offset = a->base_offset;
    d.rounds = a->rounds;
    const long long ss = hp, sh = static_cast<long long>(a->seq) * hp, sb = sh * a->slices;
    rgo_tensor4 tq{ds[0], sb, sh, ss}, tk{ds[1], sb, sh, ss}, tv{ds[2], sb, sh, ss}, to{ds[3], sb, sh, ss};
    int rc = rgo_attn_fwd(&d, &tq, &tk, &tv, dbits, bits_bytes, &to, nullptr, nullptr);
    if (rc != RGO_OK) return rc;
    unpad_to_f32<<<blocks_for(rows * hd), 256>>>(ds[3], f, rows, hd, hp);
    RGO_TRY(cudaGetLastError(), "attention");
    RGO_TRY(cudaMemcpy(h_o, f, rows * hd * 4, cudaMemcpyDeviceToHost), "attention");
    return RGO_OK;
}

int rgo_mask_save(const char* path, const rgo_mask_desc* d, float keep_prob, const uint8_t* h_bits,
                  uint64_t bytes) {
    if (!path || !d || (!h_bits && bytes)) return set_error(RGO_EINVAL, "save_mask: null argument");
    uint8_t hdr[40];
    std::memcpy(hdr, "RNGM", 4);
    put(hdr + 4, 1, 2);
    put(hdr + 6, d->rounds, 2);
    put(hdr + 8, d->batch, 4);
    put(hdr + 12, d->heads, 4);
    put(hdr + 16, d->seq, 4);
    put(hdr + 20, d->seed, 8);
    put(hdr + 28, d->base_offset, 8);
    uint32_t pb;
    std::memcpy(&pb, &keep_prob, 4);
    put(hdr + 36, pb, 4);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
    if (!f) return set_error(RGO_EIO, "save_mask: cannot open %s", path);
    if (std::fwrite(hdr, 1, 40, f.get()) != 40 || std::fwrite(h_bits, 1, bytes, f.get()) != bytes)
        return set_error(RGO_EIO, "save_mask: write failed for %s", path);
    return RGO_OK;
}

int rgo_mask_load(const char* path, rgo_mask_desc* d, float* keep_prob, uint8_t* h_bits, uint64_t capacity,
                  uint64_t* bytes) {
    if (!path || !d) return set_error(RGO_EINVAL, "load_mask: null argument");
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), &std::fclose);
    if (!f) return set_error(RGO_EIO, "load_mask: cannot open %s", path);
    uint8_t hdr[40];
    if (std::fread(hdr, 1, 40, f.get()) != 40) return set_error(RGO_EIO, "load_mask: truncated header in %s", path);
    if (std::memcmp(hdr, "RNGM", 4) != 0) return set_error(RGO_EIO, "load_mask: bad magic in %s", path);
    if (get(hdr + 4, 2) != 1) return set_error(RGO_EIO, "load_mask: unsupported version in %s", path);
    rgo_mask_desc m{};
    m.rounds = static_cast<uint32_t>(get(hdr + 6, 2));
    m.batch = static_cast<uint32_t>(get(hdr + 8, 4));
    m.heads = static_cast<uint32_t>(get(hdr + 12, 4));
    m.seq = static_cast<uint32_t>(get(hdr + 16, 4));
    m.seed = get(hdr + 20, 8);
    m.base_offset = get(hdr + 28, 8);
    const uint32_t pb = static_cast<uint32_t>(get(hdr + 36, 4));
    float kp;
    std::memcpy(&kp, &pb, 4);
    const uint64_t n = static_cast<uint64_t>(m.batch) * m.heads * m.seq * static_cast<uint64_t>(m.seq);
    if (n == 0) return set_error(RGO_EINVAL, "mask layout has zero elements");
    if (m.rounds < 1 || m.rounds > 16) return set_error(RGO_EIO, "load_mask: rounds out of range in %s", path);
    rgo_keep_threshold(kp, &m.threshold, nullptr);
    const uint64_t need = (n + 7) / 8;
    *d = m;
    if (keep_prob) *keep_prob = kp;
    if (bytes) *bytes = need;
    if (!h_bits) return RGO_OK;
    if (capacity < need) return set_error(RGO_EINVAL, "load_mask: buffer needs %llu bytes",
                                          static_cast<unsigned long long>(need));
    if (std::fread(h_bits, 1, need, f.get()) != need)
        return set_error(RGO_EIO, "load_mask: truncated payload in %s", path);
    if ((n & 7) && (h_bits[need - 1] >> (n & 7)) != 0)
        return set_error(RGO_EIO, "load_mask: nonzero padding bits in %s", path);
    return RGO_OK;
}

uint64_t rgo_fnv1a64(const uint8_t* h_data, uint64_t n) {
    // FNV-1a-64 (offset 0xcbf29ce484222325, prime 0x100000001b3): the checksum the
    // golden mask fixtures carry (tests/golden/golden.json).
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) h = (h ^ h_data[i]) * 0x100000001b3ull;
    return h;
}

}  // extern "C"
