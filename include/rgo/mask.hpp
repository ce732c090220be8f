// rgo/mask.hpp -- drop-in for proj/include/rgo/mask.hpp.  Layout, threshold
// and index arithmetic are the reference's; generate_mask runs K1 on the GPU
// (rgo_generate_mask_host; `workers` selects how many GPUs share the work --
// the bytes never depend on it), keep_bit_direct uses the GPU philox_block,
// and the RNGM file format is read/written by the C ABI.
#pragma once

#include <cmath>
#include <cstdint>
#include <filesystem>
#include <stdexcept>
#include <utility>
#include <vector>

#include "rgo/philox.hpp"

namespace rgo {

struct MaskLayout {
    uint32_t batch = 1;
    uint32_t heads = 1;
    uint32_t seq = 1;
    uint64_t seed = 0;
    uint64_t base_offset = 0;

    uint64_t elem_count() const { return uint64_t{batch} * heads * seq * uint64_t{seq}; }

    uint64_t linear_index(uint32_t b, uint32_t h, uint32_t i, uint32_t j) const {
        if (b >= batch || h >= heads || i >= seq || j >= seq)
            throw std::invalid_argument("mask index out of range");
        return ((uint64_t{b} * heads + h) * seq + i) * seq + j;
    }

    PhiloxKey key() const { return PhiloxKey{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)}; }

    void validate() const {
        if (elem_count() == 0) throw std::invalid_argument("mask layout has zero elements");
    }
};

struct KeepThreshold {
    float keep_prob = 1.0f;

    explicit KeepThreshold(double p) {
        uint64_t t;
        detail::check(rgo_keep_threshold(p, &t, &keep_prob));
    }
    uint64_t threshold() const {
        uint64_t t = 0;
        rgo_keep_threshold(keep_prob, &t, nullptr);
        return t;
    }
    bool keeps(uint32_t word) const { return word < threshold(); }
};

/// (counter, lane) deciding element `linear_index` (mask.hpp:72-85).
inline std::pair<PhiloxCounter, int> element_source(const MaskLayout& layout, uint64_t linear_index) {
    if (linear_index >= layout.elem_count())
        throw std::invalid_argument("element_source: linear index out of range");
    const uint64_t ctr = layout.base_offset + (linear_index >> 2);
    return {PhiloxCounter{static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), 0, 0},
            static_cast<int>(linear_index & 3)};
}

inline bool keep_bit_direct(const MaskLayout& layout, const KeepThreshold& thr, int rounds, uint64_t linear_index) {
    const auto src = element_source(layout, linear_index);
    return thr.keeps(philox_block(layout.key(), src.first, rounds).word(src.second));
}

struct DropoutMask {
    MaskLayout layout;
    float keep_prob = 1.0f;
    uint32_t rounds = 7;
    std::vector<uint8_t> bits;  // 1 = keep, LSB-first

    bool bit(uint32_t b, uint32_t h, uint32_t i, uint32_t j) const {
        const uint64_t idx = layout.linear_index(b, h, i, j);
        return (bits[idx >> 3] >> (idx & 7)) & 1u;
    }
};

namespace detail {
inline rgo_mask_desc to_desc(const MaskLayout& l, uint64_t threshold, int rounds) {
    rgo_mask_desc d{};
    d.batch = l.batch;
    d.heads = l.heads;
    d.seq = l.seq;
    d.rounds = static_cast<uint32_t>(rounds < 0 ? 0 : rounds);
    d.seed = l.seed;
    d.base_offset = l.base_offset;
    d.threshold = threshold;
    return d;
}
}  // namespace detail

inline DropoutMask generate_mask(const MaskLayout& layout, const KeepThreshold& thr, int rounds,
                                 unsigned workers = 0) {
    layout.validate();
    if (rounds < 1 || rounds > 16) throw std::invalid_argument("generate_mask: rounds must be in [1,16]");
    const rgo_mask_desc d = detail::to_desc(layout, thr.threshold(), rounds);
    DropoutMask m;
    m.layout = layout;
    m.keep_prob = thr.keep_prob;
    m.rounds = static_cast<uint32_t>(rounds);
    const uint64_t n = layout.elem_count();
    if (n > (uint64_t{1} << 36)) detail::check(rgo_generate_mask_host(&d, nullptr, 0, 0));  // guard message
    m.bits.assign((n + 7) / 8, 0);
    detail::check(rgo_generate_mask_host(&d, m.bits.data(), m.bits.size(), workers));
    return m;
}

inline bool mask_bit(const DropoutMask& mask, uint32_t b, uint32_t h, uint32_t i, uint32_t j) {
    return mask.bit(b, h, i, j);
}

inline void save_mask(const DropoutMask& mask, const std::filesystem::path& path) {
    const rgo_mask_desc d = detail::to_desc(mask.layout, 0, static_cast<int>(mask.rounds));
    detail::check(rgo_mask_save(path.string().c_str(), &d, mask.keep_prob, mask.bits.data(), mask.bits.size()));
}

inline DropoutMask load_mask(const std::filesystem::path& path) {
    rgo_mask_desc d{};
    float kp = 0;
    uint64_t need = 0;
    detail::check(rgo_mask_load(path.string().c_str(), &d, &kp, nullptr, 0, &need));
    DropoutMask m;
    m.bits.resize(need);
    detail::check(rgo_mask_load(path.string().c_str(), &d, &kp, m.bits.data(), m.bits.size(), &need));
    m.layout = MaskLayout{d.batch, d.heads, d.seq, d.seed, d.base_offset};
    m.keep_prob = kp;
    m.rounds = d.rounds;
    return m;
}

}  // namespace rgo
