"""Pin the CPU oracle to the reference: every golden vector frozen from the
reference package (tests/golden/make_golden.py) must be reproduced exactly.

CPU-only (no GPU marker). Mirrors the reference's own KAT / oracle-equivalence
tests (reference pkg/tests/test_generators.py:86-152, test_brownian.py:120-190).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import ALGS

M32 = 0xFFFFFFFF


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class TestKnownAnswers:
    def test_philox(self, oracle, golden):
        for ctr, key, out in golden["philox_kat"]:
            assert oracle.philox_block(key, ctr) == tuple(out)

    def test_philox_published_random123(self, oracle):
        # Random123 kat_vectors (reference tests/test_generators.py:33-40)
        assert oracle.philox_block((0, 0), (0, 0, 0, 0)) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)

    def test_threefry(self, oracle, golden):
        for ctr, key, out in golden["threefry_kat_20"]:
            assert oracle.threefry_block(key, ctr) == tuple(out)
        for ctr, key, out in golden["threefry_kat_13"]:
            assert oracle.threefry_block(key, ctr, rounds=13) == tuple(out)

    def test_squares(self, oracle, golden):
        for seed, key, words in golden["squares_kat"]:
            assert oracle.squares_key(seed) == key
            assert [oracle.squares_round(key, c) for c in range(3)] == words

    def test_tyche(self, oracle, golden):
        kat = golden["tyche_kat"]
        st = oracle.tyche_init(kat["seed"], kat["ctr"])
        assert list(st) == kat["state"]
        words = []
        for _ in range(4):
            st = oracle.tyche_mix(st)
            words.append(st[1])
        assert words == kat["words"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_stream_seed42(self, oracle, golden, alg):
        assert oracle.stream_words(alg, 42, 0, 8).tolist() == golden["stream_seed42"][alg]


class TestVectorCiphers:
    def test_random_blocks(self, oracle, golden_arrays):
        c, k = golden_arrays["blk_ctr"], golden_arrays["blk_key"]
        for i in range(0, 256, 7):
            ctr = tuple(int(x) for x in c[:, i])
            assert oracle.philox_block((int(k[0, i]), int(k[1, i])), ctr) == tuple(int(x) for x in golden_arrays["blk_philox"][:, i])
            assert oracle.threefry_block(tuple(int(x) for x in k[:, i]), ctr) == tuple(int(x) for x in golden_arrays["blk_threefry"][:, i])
            assert oracle.tyche_mix(ctr) == tuple(int(x) for x in golden_arrays["blk_tyche_state"][:, i])

    def test_squares_blocks(self, oracle, golden_arrays):
        for i in range(256):
            assert oracle.squares_round(int(golden_arrays["blk_sq_key"][i]), int(golden_arrays["blk_sq_ctr"][i])) == int(golden_arrays["blk_squares"][i])
            assert oracle.squares_key(int(golden_arrays["blk_sq_seeds"][i])) == int(golden_arrays["blk_sq_keys_of_seeds"][i])


class TestStreams:
    def test_cfg1(self, oracle, golden):
        w = oracle.stream_words("philox", 42, 0, 2**20)
        assert sha(w) == golden["cfg1"]["sha256"]
        assert int(w[0]) == golden["cfg1"]["first"] and int(w[-1]) == golden["cfg1"]["last"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_stream_digests(self, oracle, golden, golden_arrays, alg):
        for i, (s, c) in enumerate(golden["stream_pairs"]):
            w = oracle.stream_words(alg, s, c, 65536 + 3)
            assert sha(w) == golden["stream_digests"][alg][i]
            assert np.array_equal(w[:1027], golden_arrays[f"stream_{alg}_{i}"])

    @pytest.mark.parametrize("alg", ALGS)
    def test_block_counter_wrap(self, oracle, golden_arrays, alg):
        ref = golden_arrays[f"wrap_{alg}"]
        if alg == "tyche":
            # Tyche's block counter is a position tally only (generators.py:302-305)
            w = oracle.stream_words(alg, 5, 6, 200)
        else:
            w = oracle.stream_words(alg, 5, 6, 200, block_ctr=2**32 - 3)
        assert np.array_equal(w, ref)

    @pytest.mark.parametrize("alg", ["philox", "threefry"])
    def test_lane_offset(self, oracle, alg):
        full = oracle.stream_words(alg, 7, 1, 64)
        for lane in range(4):
            assert np.array_equal(oracle.stream_words(alg, 7, 1, 30, block_ctr=2, lane=lane), full[8 + lane: 38 + lane])

    def test_tyche_state_roundtrip(self, oracle):
        full = oracle.stream_words("tyche", 77, 3, 1000)
        st = oracle.tyche_init(77, 3)
        a, st = oracle.stream_words("tyche", 77, 3, 400, tyche_state=st)
        b, st = oracle.stream_words("tyche", 77, 3, 600, tyche_state=st)
        assert np.array_equal(np.concatenate([a, b]), full)

    def test_panel_digest(self, oracle, golden):
        h = hashlib.sha256()
        for alg in ALGS:
            for s, c in golden["panel"]["pairs"]:
                h.update(oracle.stream_words(alg, s, c, golden["panel"]["words"]).astype("<u4").tobytes())
        assert h.hexdigest() == golden["panel"]["sha256"]


class TestDistributions:
    @pytest.mark.parametrize("alg", ALGS)
    def test_uniform_f32(self, oracle, golden, golden_arrays, alg):
        assert sha(oracle.uniform_f32(alg, 42, 0, 2**20)) == golden["uniform_f32_2p20"][alg]
        assert sha(oracle.words_to_f32(oracle.stream_words(alg, 42, 0, 2**20))) == golden["uniform_f32_2p20"][alg]
        assert np.array_equal(oracle.uniform_f32(alg, 99, 2, 1029), golden_arrays[f"uf32_{alg}"])

    @pytest.mark.parametrize("alg", ALGS)
    def test_uniform_f64(self, oracle, golden, golden_arrays, alg):
        assert sha(oracle.uniform_f64(alg, 42, 0, 2**19)) == golden["uniform_f64_2p19"][alg]
        assert np.array_equal(oracle.uniform_f64(alg, 99, 2, 1029), golden_arrays[f"uf64_{alg}"])

    @pytest.mark.parametrize("alg", ALGS)
    def test_normal2(self, oracle, golden_arrays, alg):
        z0, z1 = oracle.normal2(alg, 42, 0, 4099)
        # glibc libm, as CPython's math module: bit-identical to the reference's
        # scalar normal2 (distributions.py:72-81)
        assert np.array_equal(z0, golden_arrays[f"n2scalar_{alg}"][:, 0])
        assert np.array_equal(z1, golden_arrays[f"n2scalar_{alg}"][:, 1])
        # the reference's bulk normal2_array (numpy SIMD libm, distributions.py:110-120)
        # differs from its own scalar path by <= 2 ulp(max(|z|, 1))
        for got, ref in ((z0, golden_arrays[f"n2bulk_{alg}_z0"]), (z1, golden_arrays[f"n2bulk_{alg}_z1"])):
            tol = 2 * np.spacing(np.maximum(np.abs(ref), 1.0))
            assert np.all(np.abs(got - ref) <= tol)


class TestPrefixWords:
    @pytest.mark.parametrize("alg", ALGS)
    def test_arange(self, oracle, golden, alg):
        w = oracle.prefix_words_arange(alg, 0, 2**16, 0, 256)
        assert sha(w) == golden["prefix_arange_2p16_256"][alg]
        assert np.array_equal(w, oracle.prefix_words(alg, np.arange(2**16, dtype=np.uint64), 0, 256))

    @pytest.mark.parametrize("alg", ALGS)
    def test_random_streams(self, oracle, golden_arrays, alg):
        seeds, ctrs = golden_arrays["prefix_seeds"], golden_arrays["prefix_ctrs"]
        for nw in (1, 4, 7, 19):
            assert np.array_equal(oracle.prefix_words(alg, seeds, ctrs, nw), golden_arrays[f"prefix_{alg}_{nw}"])
        assert np.array_equal(oracle.prefix_words(alg, seeds, 9, 12), golden_arrays[f"prefix_{alg}_scalarctr"])


class TestBrownian:
    @pytest.mark.parametrize("alg", ALGS)
    def test_checksum_1000x100(self, oracle, golden, alg):
        st = oracle.run_sim(alg, 1000, 100)
        assert f"{oracle.brownian_checksum(*st):016x}" == golden["brownian_1000x100"][alg]

    def test_checksum_acceptance_c6(self, oracle, golden):
        st = oracle.run_sim("philox", 100_000, 1000)
        assert f"{oracle.brownian_checksum(*st):016x}" == golden["brownian_1e5x1e3_philox"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_cases_bit_exact(self, oracle, golden, golden_arrays, alg):
        for key, case in golden["brownian_cases"].items():
            if not key.endswith("_" + alg):
                continue
            name = key[: -len(alg) - 1]
            cfg = dict(case["cfg"])
            n, steps = cfg["n_particles"], cfg["steps"]
            kw = dict(dt=cfg.get("dt", 0.01), gamma=cfg.get("gamma", 0.1), mass=cfg.get("mass", 1.0),
                      init_ctr=cfg.get("init_counter", 0))
            init = oracle.brownian_init(alg, n, kw["init_ctr"])
            for f, a in zip(("x", "y", "vx", "vy"), init):
                assert np.array_equal(a, golden_arrays[f"bw_{name}_{alg}_init_{f}"])
            st = oracle.run_sim(alg, n, steps, **kw)
            for f, a in zip(("x", "y", "vx", "vy"), st):
                assert np.array_equal(a, golden_arrays[f"bw_{name}_{alg}_{f}"])
            assert f"{oracle.brownian_checksum(*st):016x}" == case["checksum"]

    def test_split_steps_equal_straight(self, oracle):
        a = oracle.run_sim("philox", 50, 20)
        st = oracle.brownian_init("philox", 50)
        oracle.brownian_steps("philox", st, 1, 7)
        oracle.brownian_steps("philox", st, 8, 13)
        for u, v in zip(a, st):
            assert np.array_equal(u, v)


class TestFnv:
    def test_vectors(self, oracle, golden):
        assert oracle.fnv1a64(b"") == golden["fnv"]["empty"]
        assert oracle.fnv1a64(bytes(40)) == golden["fnv"]["zero40"]
        assert oracle.fnv1a64(bytes(range(256)) * 3) == golden["fnv"]["bytes0_255x3"]


class TestBatteryHostFormulas:
    """stats.py's statistic -> p-value -> verdict arithmetic, fed with byte
    histograms of oracle-generated words, reproduces the reference's reports."""

    def test_blob_reports(self, oracle, golden):
        import numpy as np

        from paper_2310_19925_b200 import stats as st

        blob = oracle.stream_words("squares", 3, 1, 100_003).astype("<u4").tobytes()[:400_010]
        counts = np.bincount(np.frombuffer(blob, np.uint8), minlength=256)
        assert st.report_to_dict(st.monobit_from_counts(counts)) == golden["blob_tests"]["monobit"]
        assert st.report_to_dict(st.chi_square_from_counts(counts)) == golden["blob_tests"]["chi_square_bytes"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_battery_stream_reports(self, oracle, golden, alg):
        import numpy as np

        from paper_2310_19925_b200 import stats as st

        words = oracle.stream_words(alg, st.DEFAULT_BATTERY_SEED, 0, 16 * 2**20 // 4)
        counts = np.bincount(words.view(np.uint8), minlength=256)
        ref = golden["battery_16MiB"][alg]
        assert st.report_to_dict(st.monobit_from_counts(counts)) == ref[0]
        assert st.report_to_dict(st.chi_square_from_counts(counts)) == ref[1]

    def test_classify_p_bands(self):
        from paper_2310_19925_b200 import stats as st

        assert st.classify_p(0.5) is st.Verdict.PASS
        assert st.classify_p(1e-5) is st.Verdict.SUSPICIOUS
        assert st.classify_p(1 - 1e-5) is st.Verdict.SUSPICIOUS
        assert st.classify_p(1e-7) is st.Verdict.FAIL
        assert st.classify_p(1 - 1e-7, folded=True) is st.Verdict.PASS
        assert st.classify_p(float("nan")) is st.Verdict.FAIL


def test_oracle_fullsize_cfg1_digests_match_reference():
    """The oracle's streamed digests over all 2^30 values of configs[1] equal the
    digests of the reference package's own outputs (make_golden_r2.py) — the
    oracle is pinned at full size, not only on short vectors."""
    import json

    from conftest import GOLDEN_DIR
    from oracle import oracle as orc

    ref = json.loads((GOLDEN_DIR / "golden_r2.json").read_text())["cfg1_fullsize"]["values"]
    for alg in ("philox", "squares"):
        assert f"{orc.digest_stream(alg, 42, 0, 0, 1 << 30, as_f32=True):016x}" == ref[alg], alg
    assert f"{orc.digest_prefix('tyche', 0, 1 << 22, 0, 256, as_f32=True):016x}" == ref["tyche"]


def test_oracle_digest_matches_numpy_definition():
    from oracle import oracle as orc
    from paper_2310_19925_b200 import sharding

    for alg in ("philox", "threefry", "squares"):
        w = orc.stream_words(alg, 9, 4, 5000)
        assert orc.digest_stream(alg, 9, 4, 0, 5000) == sharding.digest_words_np(w, 0)
        assert orc.digest_stream(alg, 9, 4, 1001, 3999, 1001) == sharding.digest_words_np(w[1001:], 1001)
        f = orc.words_to_f32(w).view(np.uint32)
        assert orc.digest_stream(alg, 9, 4, 0, 5000, as_f32=True) == sharding.digest_words_np(f, 0)
    w = orc.prefix_words_arange("tyche", 3, 100, 1, 256)
    assert orc.digest_prefix("tyche", 3, 100, 1, 256, 77) == sharding.digest_words_np(w.reshape(-1), 77)


def test_oracle_normal2_error_zero_on_itself():
    from oracle import oracle as orc

    z0, z1 = orc.normal2("threefry", 5, 2, 10_000)
    e = orc.normal2_error("threefry", 5, 2, 0, z0, z1)
    assert e == {"max_units": 0.0, "max_rel_ulps": 0.0, "over_tol": 0}
    z0[7] = np.nextafter(z0[7], np.inf)
    assert orc.normal2_error("threefry", 5, 2, 0, z0, z1)["max_units"] > 0
