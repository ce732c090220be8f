// rgo/philox.hpp -- drop-in for proj/include/rgo/philox.hpp (same names and
// signatures).  philox_block / philox_round run on the B200 through the C ABI
// (rgo_philox_blocks_host); bump_key / advance are the counter arithmetic of
// philox.hpp:65-80 and stay host integer helpers.
#pragma once

#include <cstdint>

#include "rgo/status.hpp"

namespace rgo {

struct PhiloxKey {
    uint32_t k0 = 0;
    uint32_t k1 = 0;
    friend bool operator==(const PhiloxKey&, const PhiloxKey&) = default;
};

struct PhiloxCounter {
    uint32_t c0 = 0;  // least significant
    uint32_t c1 = 0;
    uint32_t c2 = 0;
    uint32_t c3 = 0;
    friend bool operator==(const PhiloxCounter&, const PhiloxCounter&) = default;
};

struct PhiloxBlock {
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
    uint32_t word(int lane) const {
        const uint32_t w[4] = {w0, w1, w2, w3};
        return w[lane & 3];
    }
    friend bool operator==(const PhiloxBlock&, const PhiloxBlock&) = default;
};

/// R-round Philox-4x32 keyed permutation on the GPU (philox.hpp:84-96);
/// std::invalid_argument unless 1 <= rounds <= 16.
inline PhiloxBlock philox_block(const PhiloxKey& key, const PhiloxCounter& counter, int rounds) {
    const uint32_t k[2] = {key.k0, key.k1};
    const uint32_t c[4] = {counter.c0, counter.c1, counter.c2, counter.c3};
    const int32_t r = rounds;
    uint32_t w[4];
    detail::check(rgo_philox_blocks_host(k, c, &r, w, 1));
    return PhiloxBlock{w[0], w[1], w[2], w[3]};
}

/// One S-P round (philox.hpp:54-62) = philox_block with a single round.
inline PhiloxCounter philox_round(const PhiloxCounter& s, const PhiloxKey& key) {
    const PhiloxBlock b = philox_block(key, s, 1);
    return PhiloxCounter{b.w0, b.w1, b.w2, b.w3};
}

/// Weyl key step (philox.hpp:65-67).
inline PhiloxKey bump_key(const PhiloxKey& key) {
    return PhiloxKey{key.k0 + 0x9E3779B9u, key.k1 + 0xBB67AE85u};
}

/// 128-bit counter += n, carrying c0 -> c1 -> c2 -> c3 (philox.hpp:70-80).
inline PhiloxCounter advance(PhiloxCounter c, uint64_t n) {
    uint32_t add_lo = static_cast<uint32_t>(n), add_hi = static_cast<uint32_t>(n >> 32);
    const uint32_t lo = c.c0 + add_lo;
    if (lo < add_lo) ++add_hi;  // uint32 wrap of the carry, as in the reference
    c.c0 = lo;
    const uint32_t mid = c.c1 + add_hi;
    const bool carry = mid < add_hi;
    c.c1 = mid;
    if (carry && ++c.c2 == 0) ++c.c3;
    return c;
}

}  // namespace rgo
