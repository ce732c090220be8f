// C++ parity tests for the drop-in headers (include/rgo/*.hpp over the C ABI).
// They restate the reference's own unit tests (proj/tests/test_philox.cpp,
// test_mask.cpp, test_attention.cpp, test_workload.cpp) against the GPU-backed
// API, with a minimal harness (Catch2 is not available here).  Exit code 0
// iff every check passes; exit 77 = no CUDA device (skipped).
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>

#include "rgo/mask.hpp"
#include "rgo/philox.hpp"
#include "rgo/ref_attention.hpp"
#include "rgo/workload.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                 \
    do {                                                                            \
        if (cond) {                                                                 \
            ++g_pass;                                                               \
        } else {                                                                    \
            ++g_fail;                                                               \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);             \
        }                                                                           \
    } while (0)
template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

using namespace rgo;

static void test_philox() {  // test_philox.cpp
    CHECK(philox_round({0, 0, 0, 0}, {0, 0}) == (PhiloxCounter{0, 0, 0, 0}));
    CHECK(philox_round({1, 0, 0, 0}, {0, 0}) == (PhiloxCounter{0, 0, 0, 0xD2511F53u}));
    CHECK(bump_key({0xFFFFFFFFu, 0xFFFFFFFFu}) == (PhiloxKey{0x9E3779B8u, 0xBB67AE84u}));
    CHECK(philox_block({0, 0}, {0, 0, 0, 0}, 10) == (PhiloxBlock{0x6627e8d5u, 0xe169c58du, 0xbc57ac4cu, 0x9b00dbd8u}));
    CHECK(philox_block({0xFFFFFFFFu, 0xFFFFFFFFu}, {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, 10) ==
          (PhiloxBlock{0x408f276du, 0x41c83b0eu, 0xa20bc7c6u, 0x6d5451fdu}));
    CHECK(philox_block({0, 0}, {0, 0, 0, 0}, 1) == (PhiloxBlock{0, 0, 0, 0}));
    CHECK(throws<std::invalid_argument>([] { philox_block({0, 0}, {0, 0, 0, 0}, 0); }));
    CHECK(throws<std::invalid_argument>([] { philox_block({0, 0}, {0, 0, 0, 0}, 17); }));
    CHECK(advance({0xFFFFFFFFu, 0, 0, 0}, 1) == (PhiloxCounter{0, 1, 0, 0}));
    CHECK(advance({0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0}, 1) == (PhiloxCounter{0, 0, 0, 1}));
    CHECK(advance({0, 0, 0, 0}, 0x1'0000'0005ull) == (PhiloxCounter{5, 1, 0, 0}));
}

static void test_mask() {  // test_mask.cpp
    MaskLayout l;
    l.heads = 2;
    l.seq = 4;
    auto [c7, l7] = element_source(l, 7);
    CHECK(c7 == (PhiloxCounter{1, 0, 0, 0}) && l7 == 3);
    CHECK(throws<std::invalid_argument>([&] { element_source(l, 32); }));
    CHECK(KeepThreshold(0.9).threshold() == 3865470464ull);
    CHECK(KeepThreshold(1.0).threshold() == (uint64_t{1} << 32));
    CHECK(throws<std::invalid_argument>([] { KeepThreshold(1.1); }));

    MaskLayout e{2, 3, 16, 99, 0};
    const DropoutMask ones = generate_mask(e, KeepThreshold(1.0), 7);
    const DropoutMask zeros = generate_mask(e, KeepThreshold(0.0), 7);
    bool all = true;
    for (uint32_t b = 0; b < 2; ++b)
        for (uint32_t h = 0; h < 3; ++h)
            for (uint32_t i = 0; i < 16; ++i)
                for (uint32_t j = 0; j < 16; ++j) all = all && mask_bit(ones, b, h, i, j) && !mask_bit(zeros, b, h, i, j);
    CHECK(all);

    MaskLayout d{2, 4, 96, 0xABCDEF0102030405ull, 12345};
    const KeepThreshold thr(0.8);
    const DropoutMask m = generate_mask(d, thr, 7);
    std::mt19937_64 gen(3);
    bool same = true;
    for (int t = 0; t < 300; ++t) {
        const uint32_t b = gen() % 2, h = gen() % 4, i = gen() % 96, j = gen() % 96;
        same = same && mask_bit(m, b, h, i, j) == keep_bit_direct(d, thr, 7, d.linear_index(b, h, i, j));
    }
    CHECK(same);

    MaskLayout w{3, 5, 97, 11, 0};
    CHECK(generate_mask(w, KeepThreshold(0.75), 7, 1).bits == generate_mask(w, KeepThreshold(0.75), 7, 8).bits);

    MaskLayout big{1, 96, 1u << 17, 0, 0};
    try {
        generate_mask(big, KeepThreshold(0.5), 7);
        CHECK(false);
    } catch (const std::invalid_argument& ex) {
        const std::string s = ex.what();
        CHECK(s.find("bytes") != std::string::npos && s.find("guard") != std::string::npos);
    }

    MaskLayout f{1, 3, 50, 31337, 77};
    const DropoutMask fm = generate_mask(f, KeepThreshold(0.9), 5);
    const auto path = std::filesystem::temp_directory_path() / "rgo_cpp_roundtrip.bin";
    save_mask(fm, path);
    const DropoutMask r = load_mask(path);
    CHECK(r.bits == fm.bits && r.layout.seed == 31337 && r.layout.base_offset == 77 && r.rounds == 5 &&
          r.keep_prob == fm.keep_prob);
    CHECK(std::filesystem::file_size(path) == 40 + (f.elem_count() + 7) / 8);
    std::filesystem::resize_file(path, std::filesystem::file_size(path) - 1);
    CHECK(throws<std::runtime_error>([&] { load_mask(path); }));
    {
        std::fstream fs(path, std::ios::in | std::ios::out | std::ios::binary);
        fs.put('X');
    }
    CHECK(throws<std::runtime_error>([&] { load_mask(path); }));
    std::filesystem::remove(path);
}

static void test_attention() {  // test_attention.cpp
    const AttentionInput one = random_attention_input(2, 1, 8, 5);
    const AttentionOutput o1 = attention_forward(one);
    bool close = true;
    for (size_t i = 0; i < one.v.size(); ++i) close = close && std::fabs(o1.o[i] - one.v[i]) <= 1e-2f * (1 + std::fabs(one.v[i]));
    CHECK(close);  // SQ = 1 => O = V (to bf16 precision)

    const AttentionInput in = random_attention_input(4, 32, 16, 77);
    const AttentionOutput plain = attention_forward(in);
    CHECK(attention_dropout_fused(in, 123, 1.0, 7) == plain);
    MaskLayout l;
    l.heads = 4;
    l.seq = 32;
    l.seed = 123;
    CHECK(attention_dropout_decoupled(in, generate_mask(l, KeepThreshold(1.0), 7), 1.0) == plain);

    const AttentionInput s = random_attention_input(2, 16, 8, 3);
    CHECK(attention_dropout_fused(s, 42, 0.9, 7) == attention_dropout_fused(s, 42, 0.9, 7));
    CHECK(!(attention_dropout_fused(s, 42, 0.9, 7) == attention_dropout_fused(s, 43, 0.9, 7)));
    CHECK(throws<std::invalid_argument>([&] { attention_dropout_fused(s, 1, 0.0, 7); }));
    MaskLayout bad;
    bad.heads = 2;
    bad.seq = 8;
    CHECK(throws<std::invalid_argument>([&] { attention_dropout_decoupled(s, generate_mask(bad, KeepThreshold(0.9), 7), 0.9); }));

    int eq = 0;
    const auto res = run_equiv_suite(default_equiv_grid());
    for (const auto& r : res) eq += r.bitwise_equal;
    CHECK(res.size() == 16 && eq == 16);  // acceptance criterion 2

    const AttentionInput t = random_attention_input(3, 12, 6, 55);
    MaskLayout tl;
    tl.heads = 3;
    tl.seq = 12;
    tl.seed = 4;
    DropoutMask tm = generate_mask(tl, KeepThreshold(0.9), 7);
    const AttentionOutput base = attention_dropout_decoupled(t, tm, 0.9);
    const uint64_t idx = tl.linear_index(0, 1, 5, 7);
    tm.bits[idx >> 3] ^= static_cast<uint8_t>(1u << (idx & 7));
    const AttentionOutput tam = attention_dropout_decoupled(t, tm, 0.9);
    int rows_changed = 0;
    bool right_row = false;
    for (uint32_t ss = 0; ss < 3; ++ss)
        for (uint32_t ii = 0; ii < 12; ++ii) {
            bool diff = false;
            for (uint32_t dd = 0; dd < 6; ++dd) diff = diff || base.o[t.at(ss, ii, dd)] != tam.o[t.at(ss, ii, dd)];
            rows_changed += diff;
            right_row = right_row || (diff && ss == 1 && ii == 5);
        }
    CHECK(rows_changed == 1 && right_row);
}

static void test_workload() {  // test_workload.cpp
    WorkloadConfig u;
    u.batch = u.seq = u.heads = u.head_dim = 1;
    const auto s1 = gemm_shapes(u);
    CHECK(s1[0].m == 1 && s1[0].n == 3 && s1[0].k == 1 && s1[2].n == 4 && s1[3].k == 4);
    const auto g = gemm_shapes(workload_preset("gpt3"));
    CHECK(g[0].m == 2048 && g[0].n == 36864 && g[0].k == 12288);
    CHECK(attention_work(workload_preset("llama2")).mma_flops == 549755813888ull);
    CHECK(rng_elements(workload_preset("gpt3")) == 402653184ull);
    const auto l7 = gemm_shapes(workload_preset("llama2_7b"));
    CHECK(l7[2].n == 22016 && l7[3].k == 11008 && l7[0].m == 16384);
    CHECK(throws<std::invalid_argument>([] { workload_preset("nope"); }));
}

int main() {
    if (rgo_device_count() == 0) {
        std::printf("no CUDA device: skipped (the drop-in API has no CPU fallback)\n");
        return 77;
    }
    test_philox();
    test_mask();
    test_attention();
    test_workload();
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
