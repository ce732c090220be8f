// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
// Exposes the UNMODIFIED reference implementation (header-only C++20 under
// /root/reference/proj/include/rgo, included in place -- nothing is copied)
// through a C ABI so the oracle restatement and the GPU path can be checked
// against the reference itself.  Built by oracle/Makefile into
// oracle/_ref/librgo_ref.so; used by tests/ and bench.py --impl reference.
#include <cstring>
#include <random>
#include <stdexcept>

#include "rgo/mask.hpp"
#include "rgo/philox.hpp"
#include "rgo/ref_attention.hpp"
#include "rgo/schedule.hpp"
#include "rgo/workload.hpp"

extern "C" {

int ref_philox_block(uint32_t k0, uint32_t k1, const uint32_t c[4], int rounds,
                     uint32_t out[4]) {
    try {
        const rgo::PhiloxBlock b =
            rgo::philox_block(rgo::PhiloxKey{k0, k1}, rgo::PhiloxCounter{c[0], c[1], c[2], c[3]},
                              rounds);
        out[0] = b.w0; out[1] = b.w1; out[2] = b.w2; out[3] = b.w3;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int ref_keep_threshold(double p, uint64_t* thr, float* keep_prob_f) {
    try {
        const rgo::KeepThreshold t(p);
        *thr = t.threshold();
        if (keep_prob_f) *keep_prob_f = t.keep_prob;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// generate_mask through the reference (mask.hpp:142-179), copying the bits out.
int ref_generate_mask(uint32_t batch, uint32_t heads, uint32_t seq, uint64_t seed,
                      uint64_t base_offset, double p, int rounds, unsigned workers,
                      uint8_t* out, uint64_t out_bytes) {
    try {
        rgo::MaskLayout l;
        l.batch = batch; l.heads = heads; l.seq = seq; l.seed = seed; l.base_offset = base_offset;
        const rgo::DropoutMask m = rgo::generate_mask(l, rgo::KeepThreshold(p), rounds, workers);
        if (out_bytes < m.bits.size()) return -1;
        std::memcpy(out, m.bits.data(), m.bits.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// random_attention_input (ref_attention.hpp:176-207) -> q,k,v float buffers.
void ref_random_attention_input(uint32_t slices, uint32_t seq, uint32_t head_dim, uint64_t seed,
                                float* q, float* k, float* v) {
    const rgo::AttentionInput in = rgo::random_attention_input(slices, seq, head_dim, seed);
    std::memcpy(q, in.q.data(), in.q.size() * 4);
    std::memcpy(k, in.k.data(), in.k.size() * 4);
    std::memcpy(v, in.v.data(), in.v.size() * 4);
}

static rgo::AttentionInput make_input(uint32_t slices, uint32_t seq, uint32_t head_dim,
                                      const float* q, const float* k, const float* v) {
    rgo::AttentionInput in;
    in.slices = slices; in.seq = seq; in.head_dim = head_dim;
    const size_t n = in.elems();
    in.q.assign(q, q + n); in.k.assign(k, k + n); in.v.assign(v, v + n);
    return in;
}

// mode 0 attention_forward, 1 attention_dropout_fused, 2 attention_dropout_decoupled
// (ref_attention.hpp:108-146).  Decoupled regenerates the mask with the reference's
// generate_mask (layout batch 1, heads = slices, seed, base_offset 0).
int ref_attention(uint32_t slices, uint32_t seq, uint32_t head_dim, const float* q,
                  const float* k, const float* v, int mode, uint64_t seed, uint64_t base_offset,
                  double p, int rounds, float* o) {
    try {
        const rgo::AttentionInput in = make_input(slices, seq, head_dim, q, k, v);
        rgo::AttentionOutput out;
        if (mode == 0) {
            out = rgo::attention_forward(in);
        } else if (mode == 1) {
            out = rgo::attention_dropout_fused(in, seed, p, rounds, base_offset);
        } else {
            rgo::MaskLayout l;
            l.batch = 1; l.heads = slices; l.seq = seq; l.seed = seed; l.base_offset = base_offset;
            const rgo::DropoutMask m = rgo::generate_mask(l, rgo::KeepThreshold(p), rounds);
            out = rgo::attention_dropout_decoupled(in, m, p);
        }
        std::memcpy(o, out.o.data(), out.o.size() * 4);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// attention_dropout_decoupled (ref_attention.hpp:129-146) with the caller's packed
// mask bits (layout batch 1, heads = slices): times the attention alone, without
// the generate_mask that ref_attention's mode 2 runs first.
int ref_attention_decoupled(uint32_t slices, uint32_t seq, uint32_t head_dim, const float* q,
                            const float* k, const float* v, const uint8_t* bits, uint64_t nbytes,
                            double p, int rounds, float* o) {
    try {
        const rgo::AttentionInput in = make_input(slices, seq, head_dim, q, k, v);
        rgo::DropoutMask m;
        m.layout.batch = 1; m.layout.heads = slices; m.layout.seq = seq;
        m.keep_prob = static_cast<float>(p);
        m.rounds = static_cast<uint32_t>(rounds);
        m.bits.assign(bits, bits + nbytes);
        const rgo::AttentionOutput out = rgo::attention_dropout_decoupled(in, m, p);
        std::memcpy(o, out.o.data(), out.o.size() * 4);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// gemm_shapes (workload.hpp:44-52): fills m,n,k for QKV, Proj, FFN1, FFN2.
int ref_gemm_shapes(uint32_t batch, uint32_t seq, uint32_t heads, uint32_t head_dim,
                    uint32_t ffn_factor, uint64_t mnk[12]) {
    try {
        rgo::WorkloadConfig c;
        c.batch = batch; c.seq = seq; c.heads = heads; c.head_dim = head_dim; c.ffn_factor = ffn_factor;
        const auto s = rgo::gemm_shapes(c);
        for (int i = 0; i < 4; ++i) { mnk[3 * i] = s[i].m; mnk[3 * i + 1] = s[i].n; mnk[3 * i + 2] = s[i].k; }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// The reference tests' random philox vectors, regenerated with the same
// std::mt19937_64 draws: acceptance_main.cpp:79-90 (seed 424242, R=10) and
// test_philox.cpp:98-111 (seed 1234, R = 1 + gen() % 16).  rounds_fixed=0
// selects the random-rounds form.
void ref_philox_test_vectors(uint64_t seed, int count, int rounds_fixed, uint32_t* keys,
                             uint32_t* ctrs, int32_t* rounds, uint32_t* words) {
    std::mt19937_64 gen(seed);
    for (int t = 0; t < count; ++t) {
        uint32_t c[4] = {static_cast<uint32_t>(gen()), static_cast<uint32_t>(gen()),
                         static_cast<uint32_t>(gen()), static_cast<uint32_t>(gen())};
        uint32_t k[2] = {static_cast<uint32_t>(gen()), static_cast<uint32_t>(gen())};
        const int r = rounds_fixed ? rounds_fixed : 1 + static_cast<int>(gen() % 16);
        const rgo::PhiloxBlock b =
            rgo::philox_block(rgo::PhiloxKey{k[0], k[1]}, rgo::PhiloxCounter{c[0], c[1], c[2], c[3]}, r);
        std::memcpy(keys + 2 * t, k, 8);
        std::memcpy(ctrs + 4 * t, c, 16);
        rounds[t] = r;
        words[4 * t] = b.w0; words[4 * t + 1] = b.w1; words[4 * t + 2] = b.w2; words[4 * t + 3] = b.w3;
    }
}

// The reference's timeline composition (schedule.hpp:111-136) on given kernel
// times: in = {gemm_total, attn, rng, fused} seconds, cal = {f_gemm_under_rng,
// f_rng_under_gemm, f_drop, f_carve}; out = {t_baseline, t_overlap, speedup,
// t_rng_exposed}.  Used to check the B200 calibration script's restatement.
int ref_compose_schedule(const double in[4], const double cal[4], double out[4]) {
    try {
        rgo::KernelEstimate attn, rng, fused;
        attn.runtime_s = in[1];
        rng.runtime_s = in[2];
        fused.runtime_s = in[3];
        rgo::CalibrationFactors c;
        c.f_gemm_under_rng = cal[0];
        c.f_rng_under_gemm = cal[1];
        c.f_drop = cal[2];
        c.f_carve = cal[3];
        const rgo::ScheduleEstimate e = rgo::compose_schedule(in[0], attn, rng, fused, c);
        out[0] = e.t_baseline_s;
        out[1] = e.t_overlap_s;
        out[2] = e.speedup;
        out[3] = e.t_rng_exposed_s;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

}  // extern "C"
