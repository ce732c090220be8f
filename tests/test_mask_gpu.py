"""GPU parity for K1 (csrc/rng_mask.cu) and the device Philox: bit-exact
against the reference's KATs/vectors, the reference-generated golden masks
(tests/golden, from oracle/_ref) and the live C oracle."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_philox_kats_gpu(rgo, cuda, golden):
    assert rgo.philox_block(rgo.PhiloxKey(0, 0), rgo.PhiloxCounter(0, 0, 0, 0), 10) == rgo.PhiloxBlock(
        0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    for kat in golden["philox_kats"]:
        got = rgo.philox_block(rgo.PhiloxKey(*kat["key"]), rgo.PhiloxCounter(*kat["ctr"]), kat["rounds"])
        assert tuple(got) == tuple(kat["out"])
    assert rgo.philox_round(rgo.PhiloxCounter(1, 0, 0, 0), rgo.PhiloxKey(0, 0)) == rgo.PhiloxCounter(0, 0, 0, 0xD2511F53)
    with pytest.raises(ValueError):
        rgo.philox_block(rgo.PhiloxKey(0, 0), rgo.PhiloxCounter(), 17)


@pytest.mark.parametrize("name", ["acc_r10", "unit_rr"])
def test_philox_reference_vectors_gpu(rgo, cuda, philox_vectors, name):
    got = rgo.philox_blocks(philox_vectors[name + "_keys"], philox_vectors[name + "_ctrs"],
                            philox_vectors[name + "_rounds"])
    np.testing.assert_array_equal(got, philox_vectors[name + "_words"])


def test_golden_masks_bit_exact(rgo, cuda, golden, mask_blobs):
    for m in golden["masks"]:
        lay = rgo.MaskLayout(m["batch"], m["heads"], m["seq"], m["seed"], m["base_offset"])
        mk = rgo.generate_mask(lay, rgo.KeepThreshold(m["p"]), m["rounds"])
        assert mk.bits.size == m["bytes"]
        assert f"{oracle.fnv1a64(mk.bits):016x}" == m["fnv"], m
        if m["blob"]:
            np.testing.assert_array_equal(mk.bits, mask_blobs[m["blob"]])
        # device API, odd launch shapes: same bytes
        for grid, block, smem in ((1, 32, 0), (3, 64, 0), (0, 0, 64 * 1024)):
            d = rgo.generate_mask_device(lay, rgo.KeepThreshold(m["p"]), m["rounds"], grid=grid, block=block,
                                         dyn_smem=smem)
            np.testing.assert_array_equal(d[: m["bytes"]].cpu().numpy(), mk.bits)


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_full_size_masks_match_reference(rgo, cuda, golden, which):
    """Llama2-7B (256 MiB) and GPT-3 (48 MiB) masks at R10/R7 vs the
    reference's own generate_mask (hashed in tests/golden)."""
    m = golden["big_masks"][which]
    lay = rgo.MaskLayout(m["batch"], m["heads"], m["seq"], m["seed"], m["base_offset"])
    d = rgo.generate_mask_device(lay, rgo.KeepThreshold(m["p"]), m["rounds"])
    bits = d[: m["bytes"]].cpu().numpy()
    assert f"{oracle.fnv1a64(bits):016x}" == m["fnv"]
    frac = np.unpackbits(bits[: 1 << 20]).mean()
    assert abs(frac - 0.9) < 4 * np.sqrt(0.09 / (8 << 20))


def test_random_layouts_vs_oracle(rgo, cuda):
    rng = np.random.default_rng(11)
    for _ in range(40):
        b, h, s = int(rng.integers(1, 4)), int(rng.integers(1, 6)), int(rng.integers(1, 200))
        seed = int(rng.integers(0, 2**63))
        base = int(rng.choice([0, int(rng.integers(0, 2**63)), 0xFFFFFFFF - int(rng.integers(0, 64)),
                               2**64 - int(rng.integers(1, 4096))]))
        p = float(rng.choice([0.0, 1.0, float(rng.random())]))
        rounds = int(rng.integers(1, 17))
        got = rgo.generate_mask(rgo.MaskLayout(b, h, s, seed, base), rgo.KeepThreshold(p), rounds).bits
        want = oracle.generate_mask(b, h, s, seed, base, p, rounds)
        np.testing.assert_array_equal(got, want)


def test_slice_sharding_concatenates_to_global(rgo, cuda):
    """Rank r of n takes slices [s0, s1) with base_offset + s0*SQ^2/4: the
    per-rank masks concatenate byte-exactly."""
    B, H, S = 2, 8, 256
    thr = rgo.KeepThreshold(0.9)
    full = rgo.generate_mask(rgo.MaskLayout(B, H, S, 42, 0), thr, 10).bits
    for n in (2, 4, 8):
        per = B * H // n
        parts = [rgo.generate_mask(rgo.MaskLayout(1, per, S, 42, r * per * S * S // 4), thr, 10).bits
                 for r in range(n)]
        np.testing.assert_array_equal(np.concatenate(parts), full)


def test_keep_fraction_statistics(rgo, cuda):
    # test_mask.cpp:108-122 and test_attention.cpp:121-134
    for p in (0.5, 0.8, 0.9):
        m = rgo.generate_mask(rgo.MaskLayout(1, 4, 512, 7), rgo.KeepThreshold(p), 7)
        n = 4 * 512 * 512
        f = np.unpackbits(m.bits).sum() / n
        assert abs(f - p) <= 4 * np.sqrt(p * (1 - p) / n)


def test_keep_bit_direct_gpu(rgo, cuda):
    lay = rgo.MaskLayout(2, 4, 96, 0xABCDEF0102030405, 12345)
    thr = rgo.KeepThreshold(0.8)
    m = rgo.generate_mask(lay, thr, 7)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, lay.elem_count(), 2000)
    ctrs = np.array([tuple(rgo.element_source(lay, int(i))[0]) for i in idx], np.uint32)
    keys = np.tile(np.array(tuple(lay.key()), np.uint32), (len(idx), 1))
    words = rgo.philox_blocks(keys, ctrs, 7)
    for t, i in enumerate(idx):
        direct = int(words[t, i & 3]) < thr.threshold()
        assert bool((m.bits[i >> 3] >> (i & 7)) & 1) == direct


def test_uniform_fill_matches_random_attention_input(rgo, cuda):
    import torch
    n = 8 * 512 * 64 + 3
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    h = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    for stream in (1, 2, 3):
        rgo._lib.check(rgo._lib.lib().rgo_uniform_fill(42 ^ 0xA77E, stream, n, h.data_ptr(), f.data_ptr(),
                                                       torch.cuda.current_stream().cuda_stream))
        want = oracle.uniform(42 ^ 0xA77E, stream, n)
        np.testing.assert_array_equal(f.cpu().numpy().view(np.uint32), want.view(np.uint32))
        np.testing.assert_array_equal(h.float().cpu().numpy(), torch.from_numpy(want).bfloat16().float().numpy())


@pytest.mark.parametrize("shards", [2, 3, 7])
def test_generate_mask_shards_one_device(rgo, cuda, shards):
    """rgo_generate_mask_host's multi-shard slicing (per-shard counter offsets,
    16-byte shard boundaries, ragged last shard) on one GPU: the bytes equal the
    single-shard mask and the oracle's (mask.hpp:139-141 worker independence)."""
    lay = rgo.MaskLayout(3, 5, 97, 11)
    thr = rgo.KeepThreshold(0.75)
    one = rgo.generate_mask(lay, thr, 7, workers=1).bits
    many = rgo.generate_mask(lay, thr, 7, workers=1, shards=shards).bits
    np.testing.assert_array_equal(many, one)
    np.testing.assert_array_equal(one, oracle.generate_mask(3, 5, 97, 11, 0, 0.75, 7))
