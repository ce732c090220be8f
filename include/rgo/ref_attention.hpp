// rgo/ref_attention.hpp -- drop-in for proj/include/rgo/ref_attention.hpp.
// Same types and entry points; the forward passes run the tcgen05
// flash-attention kernel (K5 decoupled / K6 fused Philox) on the GPU through
// rgo_attention_host.  Inputs are rounded to bf16 for the tensor cores, so
// outputs match the reference's fp32 loop within the BF16 tolerance (5e-3);
// fused and decoupled results are bitwise equal to each other, as in the
// reference.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "rgo/mask.hpp"

namespace rgo {

struct AttentionInput {
    uint32_t slices = 1;
    uint32_t seq = 1;
    uint32_t head_dim = 1;
    std::vector<float> q, k, v;  // row-major (slice, pos, dim), slice = b*nH + h

    size_t elems() const { return size_t{slices} * seq * head_dim; }
    size_t at(uint32_t s, uint32_t pos, uint32_t d) const { return (size_t{s} * seq + pos) * head_dim + d; }
    float scale() const { return 1.0f / std::sqrt(static_cast<float>(head_dim)); }
    void validate() const {
        if (slices < 1 || seq < 1 || head_dim < 1) throw std::invalid_argument("attention dims must be >= 1");
        if (q.size() != elems() || k.size() != elems() || v.size() != elems())
            throw std::invalid_argument("attention input shape mismatch");
    }
};

struct AttentionOutput {
    uint32_t slices = 0, seq = 0, head_dim = 0;
    std::vector<float> o;
    friend bool operator==(const AttentionOutput&, const AttentionOutput&) = default;
};

namespace detail {
inline AttentionOutput run_attention(const AttentionInput& in, int source, double p, uint64_t seed,
                                     uint64_t base_offset, int rounds, const std::vector<uint8_t>* bits) {
    in.validate();
    rgo_attn_host_desc d{};
    d.slices = in.slices;
    d.seq = in.seq;
    d.head_dim = in.head_dim;
    d.mask_source = source;
    d.keep_prob = p;
    d.seed = seed;
    d.base_offset = base_offset;
    d.rounds = static_cast<uint32_t>(rounds);
    AttentionOutput out{in.slices, in.seq, in.head_dim, std::vector<float>(in.elems())};
    detail::check(rgo_attention_host(&d, in.q.data(), in.k.data(), in.v.data(), bits ? bits->data() : nullptr,
                                     bits ? bits->size() : 0, out.o.data()));
    return out;
}
}  // namespace detail

/// softmax(Q K^T / sqrt(dH)) V (ref_attention.hpp:108-110).
inline AttentionOutput attention_forward(const AttentionInput& in) {
    return detail::run_attention(in, RGO_MASK_NONE, 1.0, 0, 0, 1, nullptr);
}

/// Dropout with Philox regenerated inside the attention kernel (:114-126).
inline AttentionOutput attention_dropout_fused(const AttentionInput& in, uint64_t seed, double p, int rounds,
                                               uint64_t base_offset = 0) {
    if (!(p > 0.0 && p <= 1.0)) throw std::invalid_argument("attention_dropout_fused: p must be in (0,1]");
    if (rounds < 1 || rounds > 16) throw std::invalid_argument("attention_dropout_fused: rounds must be in [1,16]");
    return detail::run_attention(in, RGO_MASK_PHILOX, p, seed, base_offset, rounds, nullptr);
}

/// Dropout with keep bits read from a pre-generated mask (:129-146).
inline AttentionOutput attention_dropout_decoupled(const AttentionInput& in, const DropoutMask& mask, double p) {
    if (!(p > 0.0 && p <= 1.0)) throw std::invalid_argument("attention_dropout_decoupled: p must be in (0,1]");
    in.validate();
    if (uint64_t{mask.layout.batch} * mask.layout.heads != in.slices || mask.layout.seq != in.seq)
        throw std::invalid_argument("attention_dropout_decoupled: mask layout mismatch");
    if (static_cast<float>(p) != mask.keep_prob)
        throw std::invalid_argument("attention_dropout_decoupled: p mismatch with mask");
    return detail::run_attention(in, RGO_MASK_BITS, p, 0, 0, 1, &mask.bits);
}

struct EquivCase {
    uint32_t slices, seq, head_dim;
    uint64_t seed;
    double p;
};

struct EquivResult {
    EquivCase c;
    bool bitwise_equal = false;
};

inline std::vector<EquivCase> default_equiv_grid() {
    std::vector<EquivCase> out;
    uint64_t seed = 1000;
    const uint32_t shapes[4][3] = {{1, 16, 8}, {2, 64, 32}, {4, 128, 64}, {8, 256, 64}};
    for (const auto& s : shapes)
        for (double p : {0.5, 0.8, 0.9, 0.99}) out.push_back(EquivCase{s[0], s[1], s[2], seed++, p});
    return out;
}

/// Philox-uniform synthetic inputs, generated on the GPU (:176-207).
inline AttentionInput random_attention_input(uint32_t slices, uint32_t seq, uint32_t head_dim, uint64_t seed) {
    AttentionInput in;
    in.slices = slices;
    in.seq = seq;
    in.head_dim = head_dim;
    in.q.resize(in.elems());
    in.k.resize(in.elems());
    in.v.resize(in.elems());
    detail::check(rgo_random_attention_input_host(slices, seq, head_dim, seed, in.q.data(), in.k.data(), in.v.data()));
    return in;
}

inline std::vector<EquivResult> run_equiv_suite(const std::vector<EquivCase>& cases, int rounds = 7) {
    std::vector<EquivResult> res;
    for (const EquivCase& c : cases) {
        const AttentionInput in = random_attention_input(c.slices, c.seq, c.head_dim, c.seed ^ 0xA77E);
        MaskLayout layout;
        layout.heads = c.slices;
        layout.seq = c.seq;
        layout.seed = c.seed;
        const DropoutMask mask = generate_mask(layout, KeepThreshold(c.p), rounds);
        res.push_back(EquivResult{c, attention_dropout_fused(in, c.seed, c.p, rounds) ==
                                         attention_dropout_decoupled(in, mask, c.p)});
    }
    return res;
}

}  // namespace rgo
