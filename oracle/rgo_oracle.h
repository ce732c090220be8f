/* rgo_oracle.h -- CPU oracle (TEST INFRASTRUCTURE ONLY; see rgo_oracle.c).
 * Same function set is exported by oracle/_ref/librgo_ref.so (prefix ref_)
 * built from the reference's own headers by oracle/ref_shim.cpp. */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int oracle_philox_block(uint32_t k0, uint32_t k1, const uint32_t ctr[4], int rounds,
                        uint32_t out[4]);
int oracle_keep_threshold(double p, uint64_t* thr, float* keep_prob_f);
int oracle_keep_bit_direct(uint64_t seed, uint64_t base_offset, uint64_t thr, int rounds,
                           uint64_t linear_index);
int oracle_generate_mask(uint64_t elems, uint64_t seed, uint64_t base_offset, uint64_t thr,
                         int rounds, unsigned workers, uint8_t* out, uint64_t out_bytes);
void oracle_fill_uniform(uint64_t seed, uint32_t stream, float* dst, uint64_t n);
int oracle_attention(uint32_t slices, uint32_t seq, uint32_t head_dim, const float* q,
                     const float* k, const float* v, int keep_mode, uint64_t seed,
                     uint64_t base_offset, uint64_t thr, float keep_prob_f, int rounds,
                     const uint8_t* mask_bits, uint32_t s_begin, uint32_t s_end, float* o);
uint64_t oracle_fnv1a64(const uint8_t* data, uint64_t n);

#ifdef __cplusplus
}
#endif
