/*
 * rgo_oracle.c -- CPU ORACLE for the dropout-RNG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference's CPU algorithm (/root/reference/proj/include/rgo/ headers) and is
 * used exclusively as the *checker* by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg.  The product path
 * (paper_2410_07531_b200/, include/rgo/) never links, loads or calls it.
 *
 * Parity is pinned (tests/test_oracle.py) against:
 *   - the reference's own known-answer vectors (test_philox.cpp:78-87),
 *   - the reference compiled from its own headers (oracle/_ref, built by
 *     oracle/Makefile from /root/reference/proj/include) when available,
 *   - golden fixtures generated from that build (tests/golden/, made by
 *     oracle/make_golden.py), which travel to the GPU box.
 *
 * Every function cites the reference file:line it restates.
 */
#include "rgo_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define M0 0xD2511F53u /* philox.hpp:46 */
#define M1 0xCD9E8D57u /* philox.hpp:47 */
#define W0 0x9E3779B9u /* philox.hpp:48 */
#define W1 0xBB67AE85u /* philox.hpp:49 */

/* philox.hpp:54-62 (one S-P round) and :84-96 (R rounds, R-1 key bumps). */
int oracle_philox_block(uint32_t k0, uint32_t k1, const uint32_t ctr[4], int rounds,
                        uint32_t out[4]) {
    if (rounds < 1 || rounds > 16) return -1; /* philox.hpp:86-87 */
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) { /* bump_key, philox.hpp:65-67 */
            k0 += W0;
            k1 += W1;
        }
        const uint64_t p0 = (uint64_t)M0 * c0;
        const uint64_t p1 = (uint64_t)M1 * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
    return 0;
}

/* KeepThreshold, mask.hpp:53-68: keep_prob is stored as float, then
 * threshold = llround(double(float p) * 2^32). */
int oracle_keep_threshold(double p, uint64_t* thr, float* keep_prob_f) {
    if (!(p >= 0.0 && p <= 1.0)) return -1; /* mask.hpp:57-58 */
    const float pf = (float)p;
    if (keep_prob_f) *keep_prob_f = pf;
    *thr = (uint64_t)llround((double)pf * 4294967296.0);
    return 0;
}

/* element_source + philox_block + keeps, mask.hpp:72-92. */
int oracle_keep_bit_direct(uint64_t seed, uint64_t base_offset, uint64_t thr, int rounds,
                           uint64_t linear_index) {
    const uint64_t ctr64 = base_offset + (linear_index >> 2); /* wrapping, mask.hpp:78 */
    const uint32_t ctr[4] = {(uint32_t)ctr64, (uint32_t)(ctr64 >> 32), 0u, 0u};
    uint32_t w[4];
    if (oracle_philox_block((uint32_t)seed, (uint32_t)(seed >> 32), ctr, rounds, w) != 0)
        return -1;
    return (uint64_t)w[linear_index & 3] < thr ? 1 : 0;
}

/* mask_detail::fill_byte_range, mask.hpp:111-135. */
static void fill_byte_range(uint64_t seed, uint64_t base_offset, uint64_t thr, int rounds,
                            uint64_t byte_begin, uint64_t byte_end, uint64_t n,
                            uint8_t* out) {
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (uint64_t byte = byte_begin; byte < byte_end; ++byte) {
        uint8_t acc = 0;
        for (int half = 0; half < 2; ++half) {
            const uint64_t block = byte * 2 + (uint64_t)half;
            if (block * 4 >= n) break;
            const uint64_t c = base_offset + block;
            const uint32_t ctr[4] = {(uint32_t)c, (uint32_t)(c >> 32), 0u, 0u};
            uint32_t w[4];
            oracle_philox_block(k0, k1, ctr, rounds, w);
            for (int lane = 0; lane < 4; ++lane) {
                const uint64_t idx = block * 4 + (uint64_t)lane;
                if (idx >= n) break;
                if ((uint64_t)w[lane] < thr) acc |= (uint8_t)(1u << (idx & 7));
            }
        }
        out[byte] = acc;
    }
}

typedef struct {
    uint64_t seed, base, thr, lo, hi, n;
    int rounds;
    uint8_t* out;
} fill_job;

static void* fill_thread(void* arg) {
    fill_job* j = (fill_job*)arg;
    fill_byte_range(j->seed, j->base, j->thr, j->rounds, j->lo, j->hi, j->n, j->out);
    return NULL;
}

/* generate_mask, mask.hpp:142-179: byte-aligned shards, output independent of
 * the worker count; inline when workers <= 1 or < 1024 bytes (:164-167).
 * The 2^36-bit guard (:148-155) is the caller's job (returns -2 here). */
int oracle_generate_mask(uint64_t elems, uint64_t seed, uint64_t base_offset, uint64_t thr,
                         int rounds, unsigned workers, uint8_t* out, uint64_t out_bytes) {
    if (elems == 0) return -1;
    if (rounds < 1 || rounds > 16) return -1;
    if (elems > (UINT64_C(1) << 36)) return -2;
    const uint64_t bytes = (elems + 7) / 8;
    if (out_bytes < bytes) return -1;
    if (workers <= 1 || bytes < 1024) {
        fill_byte_range(seed, base_offset, thr, rounds, 0, bytes, elems, out);
        return 0;
    }
    const uint64_t chunk = (bytes + workers - 1) / workers;
    pthread_t* th = (pthread_t*)calloc(workers, sizeof(pthread_t));
    fill_job* jobs = (fill_job*)calloc(workers, sizeof(fill_job));
    unsigned started = 0;
    for (unsigned w = 0; w < workers; ++w) {
        const uint64_t lo = (uint64_t)w * chunk;
        if (lo >= bytes) break;
        const uint64_t hi = lo + chunk < bytes ? lo + chunk : bytes;
        jobs[w] = (fill_job){seed, base_offset, thr, lo, hi, elems, rounds, out};
        pthread_create(&th[w], NULL, fill_thread, &jobs[w]);
        ++started;
    }
    for (unsigned w = 0; w < started; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
    return 0;
}

/* random_attention_input fill, ref_attention.hpp:176-207: Philox-10,
 * key = seed, counter = (block lo, block hi, stream, 0x5eed),
 * value = float(word) * (2/2^32) - 1.  Built with -ffp-contract=off so no
 * FMA contraction changes the float results (oracle/Makefile). */
void oracle_fill_uniform(uint64_t seed, uint32_t stream, float* dst, uint64_t n) {
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (uint64_t i = 0; i < n; i += 4) {
        const uint64_t block = i / 4;
        const uint32_t ctr[4] = {(uint32_t)block, (uint32_t)(block >> 32), stream, 0x5eedu};
        uint32_t w[4];
        oracle_philox_block(k0, k1, ctr, 10, w);
        for (int lane = 0; lane < 4 && i + (uint64_t)lane < n; ++lane) {
            dst[i + (uint64_t)lane] = (float)w[lane] * (2.0f / 4294967296.0f) - 1.0f;
        }
    }
}

/* attn_detail::forward_impl, ref_attention.hpp:56-92.  keep_mode:
 *   0 = no dropout (attention_forward, :108-110)
 *   1 = fused: keep bit recomputed from Philox (attention_dropout_fused, :114-126;
 *       layout_for = batch 1, heads = slices, :94-103)
 *   2 = decoupled: keep bit read from packed mask (attention_dropout_decoupled,
 *       :129-146; bit index (s*SQ + i)*SQ + j, :141-143)
 * slice range [s_begin, s_end) lets callers run a sample of slices; the
 * output pointer o is indexed globally. */
int oracle_attention(uint32_t slices, uint32_t seq, uint32_t head_dim, const float* q,
                     const float* k, const float* v, int keep_mode, uint64_t seed,
                     uint64_t base_offset, uint64_t thr, float keep_prob_f, int rounds,
                     const uint8_t* mask_bits, uint32_t s_begin, uint32_t s_end, float* o) {
    if (slices < 1 || seq < 1 || head_dim < 1) return -1;
    if (s_end > slices || s_begin > s_end) return -1;
    const float scale = 1.0f / sqrtf((float)head_dim); /* ref_attention.hpp:33 */
    const float p = keep_mode == 0 ? 1.0f : keep_prob_f;
    float* w = (float*)malloc(sizeof(float) * seq);
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#define AT(s, pos, d) (((size_t)(s) * seq + (pos)) * head_dim + (d))
    for (uint32_t s = s_begin; s < s_end; ++s) {
        for (uint32_t d = 0; d < head_dim; ++d)
            for (uint32_t i = 0; i < seq; ++i) o[AT(s, i, d)] = 0.0f;
        for (uint32_t i = 0; i < seq; ++i) {
            float row_max = -INFINITY;
            for (uint32_t j = 0; j < seq; ++j) {
                float dot = 0.0f;
                for (uint32_t d = 0; d < head_dim; ++d) dot += q[AT(s, i, d)] * k[AT(s, j, d)];
                w[j] = dot * scale;
                if (w[j] > row_max) row_max = w[j];
            }
            float denom = 0.0f;
            for (uint32_t j = 0; j < seq; ++j) {
                w[j] = expf(w[j] - row_max);
                denom += w[j];
            }
            for (uint32_t j = 0; j < seq; ++j) {
                float weight = w[j] / denom;
                if (keep_mode != 0) {
                    const uint64_t idx = ((uint64_t)s * seq + i) * seq + j;
                    int keep;
                    if (keep_mode == 1) {
                        const uint64_t c = base_offset + (idx >> 2);
                        const uint32_t ctr[4] = {(uint32_t)c, (uint32_t)(c >> 32), 0u, 0u};
                        uint32_t wd[4];
                        oracle_philox_block(k0, k1, ctr, rounds, wd);
                        keep = (uint64_t)wd[idx & 3] < thr;
                    } else {
                        keep = (mask_bits[idx >> 3] >> (idx & 7)) & 1u;
                    }
                    weight = keep ? weight / p : 0.0f;
                }
                for (uint32_t d = 0; d < head_dim; ++d) o[AT(s, i, d)] += weight * v[AT(s, j, d)];
            }
        }
    }
#undef AT
    free(w);
    return 0;
}

uint64_t oracle_fnv1a64(const uint8_t* data, uint64_t n) {
    uint64_t h = UINT64_C(0xcbf29ce484222325);
    for (uint64_t i = 0; i < n; ++i) {
        h ^= data[i];
        h *= UINT64_C(0x100000001b3);
    }
    return h;
}
