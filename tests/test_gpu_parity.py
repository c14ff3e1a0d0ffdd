"""Parity of the sm_100a CUDA path with the reference, through the C ABI.

Bar: bit-exact for every integer stream and exact float map; Box-Muller within
4 ulp(max(|z|, 1)) of the oracle (glibc libm, bit-identical to the reference's
scalar normal2 — tests/test_oracle.py). Expected values come from the golden
fixtures frozen from the reference (tests/golden) and from the CPU oracle on
the same seeded inputs. Mirrors the reference's own suites
(pkg/tests/test_generators.py, test_distributions.py, test_brownian.py).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import ALGS

pytestmark = pytest.mark.gpu

M32 = 0xFFFFFFFF
BM_ULP = 4  # Box-Muller tolerance, in ulp(max(|z|, 1))
BM_REL_ULP = 8  # and in ulps of z itself (observed: 4 over all 2^34 values of configs[3], r2z kernel)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_19925_b200 as cb

    return cb


def host(t):
    import torch

    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


class TestKnownAnswers:
    def test_block_functions(self, cb, golden):
        for ctr, key, out in golden["philox_kat"]:
            assert tuple(cb.philox_block(key, ctr)) == tuple(out)
        for ctr, key, out in golden["threefry_kat_20"]:
            assert tuple(cb.threefry_block(key, ctr)) == tuple(out)
        for ctr, key, out in golden["threefry_kat_13"]:
            assert tuple(cb.threefry_block(key, ctr, rounds=13)) == tuple(out)
        for seed, key, words in golden["squares_kat"]:
            assert cb.squares_key(seed) == key
            assert [cb.squares_round(key, c) for c in range(3)] == words
        kat = golden["tyche_kat"]
        st = cb.tyche_init(kat["seed"], kat["ctr"])
        assert list(st) == kat["state"]
        words = []
        for _ in range(4):
            w, st = cb.tyche_next(st)
            words.append(w)
        assert words == kat["words"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_stream_seed42_scalar_and_bulk(self, cb, golden, alg):
        g = cb.make_generator(alg, 42, 0)
        assert [g.next_u32() for _ in range(8)] == golden["stream_seed42"][alg]
        assert host(cb.make_generator(alg, 42, 0).words(8)).tolist() == golden["stream_seed42"][alg]

    def test_vector_ciphers(self, cb, golden_arrays):
        from paper_2310_19925_b200 import bulk

        c, k = golden_arrays["blk_ctr"], golden_arrays["blk_key"]
        assert np.array_equal(np.stack(bulk.philox4x32(*c, k[0], k[1])), golden_arrays["blk_philox"])
        assert np.array_equal(np.stack(bulk.threefry4x32(*c, *k)), golden_arrays["blk_threefry"])
        assert np.array_equal(bulk.squares32(golden_arrays["blk_sq_ctr"], golden_arrays["blk_sq_key"]),
                              golden_arrays["blk_squares"])
        assert np.array_equal(bulk.squares_keys(golden_arrays["blk_sq_seeds"]), golden_arrays["blk_sq_keys_of_seeds"])
        assert np.array_equal(np.stack(bulk.tyche_mix(*c)), golden_arrays["blk_tyche_state"])


class TestSingleStream:
    def test_cfg1_bit_exact(self, cb, golden):
        """BASELINE.json configs[0]: Philox u32 fill 2^20, seed 42, ctr 0."""
        w = host(cb.make_generator("philox", 42, 0).words(2**20))
        assert sha(w) == golden["cfg1"]["sha256"]
        assert int(w[0]) == golden["cfg1"]["first"] and int(w[-1]) == golden["cfg1"]["last"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_stream_digests(self, cb, golden, golden_arrays, alg):
        for i, (s, c) in enumerate(golden["stream_pairs"]):
            w = cb.make_generator(alg, s, c).words(65536 + 3, device="cpu")
            assert isinstance(w, np.ndarray) and w.dtype == np.uint32
            assert sha(w) == golden["stream_digests"][alg][i]

    @pytest.mark.parametrize("alg", ALGS)
    def test_block_counter_wrap(self, cb, golden, golden_arrays, alg):
        g = cb.make_generator(alg, 5, 6)
        g._block_ctr = 2**32 - 3
        w = host(g.words(200))
        assert np.array_equal(w, golden_arrays[f"wrap_{alg}"])
        assert g._block_ctr == golden["wrap"][alg]["block_ctr_after"]
        assert g._cache_pos == golden["wrap"][alg]["cache_pos_after"]

    @pytest.mark.parametrize("alg", ALGS)
    def test_mixed_scalar_bulk_state(self, cb, golden, alg):
        """The reference's interleaving sequence (make_golden.py state_after)."""
        g = cb.make_generator(alg, 0xFEEDFACE, 3)
        seq = [g.next_u32() for _ in range(3)]
        seq += host(g.words(130)).tolist()
        seq += [g.next_u32() for _ in range(2)]
        seq += host(g.words(1001)).tolist()
        ref = golden["state_after"][alg]
        assert sha(np.array(seq, dtype=np.uint32)) == ref["sha"]
        assert g.state_bytes().hex() == ref["state_bytes"]
        if alg == "tyche":
            assert list(g._tyche_state) == ref["tyche_state"]

    @pytest.mark.parametrize("alg", ALGS)
    @pytest.mark.parametrize("split", [0, 1, 4, 7, 3731])
    def test_serialize_restore(self, cb, oracle, alg, split):
        straight = oracle.stream_words(alg, 0x1234567, 9, 5000)
        g = cb.make_generator(alg, 0x1234567, 9)
        head = host(g.words(split))
        restored = cb.Generator.from_state_bytes(g.state_bytes())
        tail = host(restored.words(5000 - split))
        assert np.array_equal(np.concatenate([head, tail]), straight)

    @pytest.mark.parametrize("alg", ["philox", "threefry"])
    @pytest.mark.parametrize("skip", [1, 2, 3])
    def test_resume_mid_block_all_maps(self, cb, oracle, alg, skip):
        """A generator resumed mid-block fills through the 2-block kernel variant."""
        ref = oracle.stream_words(alg, 77, 5, 4 * 5000 + 16)
        for kind in ("words", "f32", "f64"):
            g = cb.make_generator(alg, 77, 5)
            [g.next_u32() for _ in range(skip)]
            if kind == "words":
                assert np.array_equal(host(g.words(4099)), ref[skip:skip + 4099])
            elif kind == "f32":
                assert np.array_equal(host(cb.uniform_f32_array(g, 4099)), oracle.words_to_f32(ref[skip:skip + 4099]))
            elif skip % 2 == 0:
                assert np.array_equal(host(cb.uniform_f64_array(g, 2049)), oracle.words_to_f64(ref[skip:skip + 4098]))
            else:
                got = host(cb.uniform_f64_array(g, 2049))
                assert np.array_equal(got, oracle.words_to_f64(ref[skip:skip + 4098]))

    @pytest.mark.parametrize("alg", ALGS)
    def test_edge_sizes(self, cb, oracle, alg):
        for n in (0, 1, 2, 3, 4, 5, 127, 128, 129, 1023, 4097):
            w = host(cb.make_generator(alg, 31337, 9).words(n))
            assert np.array_equal(w, oracle.stream_words(alg, 31337, 9, n))

    def test_negative_count_rejected(self, cb):
        with pytest.raises(ValueError):
            cb.make_generator("philox", 1, 0).words(-1)

    def test_unknown_algorithm_rejected(self, cb):
        with pytest.raises(ValueError):
            cb.make_generator("mt19937", 1, 0)


class TestDistributions:
    @pytest.mark.parametrize("alg", ALGS)
    def test_uniform_f32_f64(self, cb, golden, golden_arrays, alg):
        assert sha(host(cb.uniform_f32_array(cb.make_generator(alg, 42, 0), 2**20))) == golden["uniform_f32_2p20"][alg]
        assert sha(host(cb.uniform_f64_array(cb.make_generator(alg, 42, 0), 2**19))) == golden["uniform_f64_2p19"][alg]
        assert np.array_equal(host(cb.uniform_f32_array(cb.make_generator(alg, 99, 2), 1029)), golden_arrays[f"uf32_{alg}"])
        assert np.array_equal(host(cb.uniform_f64_array(cb.make_generator(alg, 99, 2), 1029)), golden_arrays[f"uf64_{alg}"])

    @pytest.mark.parametrize("alg", ALGS)
    def test_normal2_within_tolerance(self, cb, oracle, golden_arrays, alg):
        z0, z1 = (host(z) for z in cb.normal2_array(cb.make_generator(alg, 42, 0), 4099))
        ref = golden_arrays[f"n2scalar_{alg}"]
        for got, r in ((z0, ref[:, 0]), (z1, ref[:, 1])):
            ulps = np.abs(got - r) / np.spacing(np.maximum(np.abs(r), 1.0))
            assert ulps.max() <= BM_ULP, ulps.max()

    @pytest.mark.parametrize("alg", ALGS)
    def test_normal2_vs_reference_bulk_path(self, cb, golden_arrays, alg, record_property):
        """Against the reference's own bulk normal2_array (numpy's vectorised
        log/sqrt/cos/sin, distributions.py:110-120), not only its scalar path:
        the same absolute bound, and the relative error in ulps of z reported."""
        z0, z1 = (host(z) for z in cb.normal2_array(cb.make_generator(alg, 42, 0), 4099))
        worst_rel = 0.0
        for got, r in ((z0, golden_arrays[f"n2bulk_{alg}_z0"]), (z1, golden_arrays[f"n2bulk_{alg}_z1"])):
            assert np.all(np.abs(got - r) <= BM_ULP * np.spacing(np.maximum(np.abs(r), 1.0)))
            nz = r != 0
            worst_rel = max(worst_rel, float((np.abs(got - r)[nz] / np.spacing(np.abs(r[nz]))).max()))
        record_property("box_muller_max_rel_ulp_vs_bulk", worst_rel)
        assert worst_rel <= BM_REL_ULP, worst_rel

    def test_normal2_large_vs_oracle(self, cb, oracle):
        n = 1 << 20
        z0, z1 = (host(z) for z in cb.normal2_array(cb.make_generator("philox", 42, 0), n))
        r0, r1 = oracle.normal2("philox", 42, 0, n)
        for got, r in ((z0, r0), (z1, r1)):
            ulps = np.abs(got - r) / np.spacing(np.maximum(np.abs(r), 1.0))
            assert ulps.max() <= BM_ULP, ulps.max()

    @pytest.mark.parametrize("n,off", [(1, 0), (3, 0), (511, 0), (513, 0), (5 * 512 * 148 + 77, 0), (4099, 1),
                                       (2, 1)])
    def test_normal2_ragged_and_aligned(self, cb, oracle, n, off):
        """Philox Box-Muller through the warp-specialised kernel (16-byte aligned
        outputs; partial last tile, fewer pairs than one tile, more tiles than the
        grid) and through the fused kernel (outputs only 8-byte aligned)."""
        import torch

        z0 = torch.empty(n + off, dtype=torch.float64, device="cuda")[off:]
        z1 = torch.empty(n + off, dtype=torch.float64, device="cuda")[off:]
        cb.normal2_array(cb.make_generator("philox", 7, 11), n, out=(z0, z1))
        r0, r1 = oracle.normal2("philox", 7, 11, n)
        for got, r in ((host(z0), r0), (host(z1), r1)):
            assert np.all(np.abs(got - r) <= BM_ULP * np.spacing(np.maximum(np.abs(r), 1.0)))

    def test_normal2_words_edges(self, cb, oracle, record_property):
        """Box-Muller over chosen words: u1 = 1 (r = 0), u1 = 2^-53 (largest r),
        u1 next to 1 and to binade / log-table boundaries, t on and next to the
        quadrant boundaries, plus 2^22 random pairs."""
        rng = np.random.default_rng(2310)
        u_edges = [0, 1, 2, 3, 0x7FF, 1 << 20, (1 << 52) - 1, 1 << 52, (1 << 52) + 1, (1 << 53) - 1, (1 << 53) - 2,
                   (1 << 51), 3 << 50, (1 << 53) - (1 << 45), (1 << 53) - (1 << 44) - 1]
        u2_edges = [0, 1, (1 << 53) - 1] + [(k << 51) + d for k in range(4) for d in (-1, 0, 1) if (k << 51) + d >= 0]
        pairs = [(u, v) for u in u_edges for v in u2_edges]
        u_rand = rng.integers(0, 1 << 53, size=(1 << 22), dtype=np.uint64)
        v_rand = rng.integers(0, 1 << 53, size=(1 << 22), dtype=np.uint64)
        u_all = np.concatenate([np.array([p[0] for p in pairs], np.uint64), u_rand])
        v_all = np.concatenate([np.array([p[1] for p in pairs], np.uint64), v_rand])
        a = u_all << np.uint64(11) | (u_all & np.uint64(0x7FF))  # low 11 bits are dropped by the map
        b = v_all << np.uint64(11)
        w = np.empty((u_all.size, 4), np.uint32)
        w[:, 0], w[:, 1] = (a & np.uint64(0xFFFFFFFF)).astype(np.uint32), (a >> np.uint64(32)).astype(np.uint32)
        w[:, 2], w[:, 3] = (b & np.uint64(0xFFFFFFFF)).astype(np.uint32), (b >> np.uint64(32)).astype(np.uint32)
        z0, z1 = (host(z) for z in cb.words_to_normal2(w))
        r0, r1 = oracle.words_to_normal2(w)
        worst = 0.0
        for got, r in ((z0, r0), (z1, r1)):
            ulps = np.abs(got - r) / np.spacing(np.maximum(np.abs(r), 1.0))
            worst = max(worst, float(ulps.max()))
        record_property("box_muller_max_ulp", worst)
        assert worst <= BM_ULP, worst
        assert z0[0] == 0 and z1[0] == 0  # u1 == 1 -> r == 0

    @pytest.mark.parametrize("alg", ["philox", "threefry", "squares"])
    def test_normal2_long_stream_boundary(self, cb, oracle, alg):
        """configs[3] long-stream layout across a stream boundary: pair i comes
        from stream (seed, ctr0 + i div P) at pair i mod P (P = 2^32 pairs,
        2^30 for Squares), computed from an offset without the pairs before it."""
        import torch

        from paper_2310_19925_b200 import sharding

        per = sharding.pairs_per_stream(alg)
        lo, hi, seed, ctr0 = per - 5, per + 7, 42, 0xFFFFFFFF  # the stream counter wraps too
        z0 = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        z1 = torch.empty_like(z0)
        sharding.normal2_long(alg, seed, ctr0, lo, hi, z0, z1)
        words = []
        for s, off, k in sharding.stream_segments(lo, hi, per):
            bc = 4 * off if alg == "squares" else off
            words.append(oracle.stream_words(alg, seed, (ctr0 + s) & M32, 4 * k, block_ctr=bc))
        r0, r1 = oracle.words_to_normal2(np.concatenate(words))
        for got, r in ((host(z0), r0), (host(z1), r1)):
            assert np.all(np.abs(got - r) <= BM_ULP * np.spacing(np.maximum(np.abs(r), 1.0)))

    def test_scalar_forms(self, cb, oracle):
        g = cb.make_generator("threefry", 12, 0)
        w = oracle.stream_words("threefry", 12, 0, 64)
        u = cb.uniform_f64(g)
        assert u == ((int(w[0]) | (int(w[1]) << 32)) >> 11) * 2.0**-53
        assert cb.range_u32(g, 6) == (int(w[2]) * 6) >> 32
        assert cb.fill_bytes(cb.make_generator("philox", 42, 0), 5) == oracle.stream_words("philox", 42, 0, 2).astype("<u4").tobytes()[:5]


class TestPrefixWords:
    @pytest.mark.parametrize("alg", ALGS)
    def test_random_streams(self, cb, golden_arrays, alg):
        from paper_2310_19925_b200 import bulk

        seeds, ctrs = golden_arrays["prefix_seeds"], golden_arrays["prefix_ctrs"]
        for nw in (1, 4, 7, 19):
            assert np.array_equal(host(bulk.prefix_words(alg, seeds, ctrs, nw)), golden_arrays[f"prefix_{alg}_{nw}"])
        assert np.array_equal(host(bulk.prefix_words(alg, seeds, 9, 12)), golden_arrays[f"prefix_{alg}_scalarctr"])

    @pytest.mark.parametrize("alg", ALGS)
    def test_arange_2p16_x256(self, cb, golden, alg):
        from paper_2310_19925_b200 import bulk

        w = host(bulk.prefix_words(alg, range(2**16), 0, 256))
        assert sha(w) == golden["prefix_arange_2p16_256"][alg]

    @pytest.mark.parametrize("alg", ALGS)
    def test_row_shapes(self, cb, oracle, alg):
        from paper_2310_19925_b200 import bulk

        # incl. 256-word rows (the compile-time-specialised kernel) with full and
        # partial warps of streams
        for n, nw in ((1, 1), (33, 8), (100, 36), (65, 128), (7, 260), (1000, 33), (1000, 256), (5, 256), (64, 256)):
            got = host(bulk.prefix_words(alg, range(1000, 1000 + n), 3, nw))
            assert np.array_equal(got, oracle.prefix_words_arange(alg, 1000, n, 3, nw))
            f = host(bulk.prefix_uniform_f32(alg, range(1000, 1000 + n), 3, nw)).reshape(-1)
            assert np.array_equal(f, oracle.words_to_f32(oracle.prefix_words_arange(alg, 1000, n, 3, nw)))

    @pytest.mark.parametrize("alg", ALGS)
    def test_prefix_uniform_f32(self, cb, oracle, alg):
        from paper_2310_19925_b200 import bulk

        got = host(bulk.prefix_uniform_f32(alg, range(4096), 0, 256))
        ref = oracle.words_to_f32(oracle.prefix_words_arange(alg, 0, 4096, 0, 256).reshape(-1)).reshape(4096, 256)
        assert np.array_equal(got, ref)

    def test_philox_block_lanes(self, cb, golden_arrays, oracle):
        from paper_2310_19925_b200 import bulk

        seeds = golden_arrays["prefix_seeds"]
        scs = golden_arrays["prefix_ctrs"].astype(np.uint64)
        got = host(bulk.philox_block_lanes(seeds, scs, 3))
        ref = oracle.prefix_words("philox", seeds, golden_arrays["prefix_ctrs"], 16)[:, 12:16]
        assert np.array_equal(got, ref)


class TestBrownian:
    @pytest.mark.parametrize("alg", ALGS)
    @pytest.mark.parametrize("mode", ["fused", "per_step"])
    def test_checksum_1000x100(self, cb, golden, alg, mode):
        r = cb.run_sim(cb.SimConfig(1000, 100, algorithm=alg, mode=mode))
        assert str(r.checksum) == golden["brownian_1000x100"][alg]

    @pytest.mark.parametrize("alg", ALGS)
    def test_cases_bit_exact(self, cb, golden, golden_arrays, alg):
        for key, case in golden["brownian_cases"].items():
            if not key.endswith("_" + alg):
                continue
            name = key[: -len(alg) - 1]
            cfg = cb.SimConfig(**case["cfg"])
            p0 = cb.init_particles(cfg)
            for f in ("x", "y", "vx", "vy"):
                assert np.array_equal(host(getattr(p0, f)), golden_arrays[f"bw_{name}_{alg}_init_{f}"])
            r = cb.run_sim(cfg)
            for f in ("x", "y", "vx", "vy"):
                assert np.array_equal(host(getattr(r.particles, f)), golden_arrays[f"bw_{name}_{alg}_{f}"]), f
            assert str(r.checksum) == case["checksum"]

    def test_acceptance_c6_shape(self, cb, golden):
        r = cb.run_sim(cb.SimConfig(100_000, 1000))
        assert str(r.checksum) == golden["brownian_1e5x1e3_philox"]

    @pytest.mark.parametrize("mode", ["fused", "per_step"])
    def test_chunked_steps_bit_exact(self, cb, oracle, mode):
        """Walks longer than the fused kernel's 256-step table, from an odd start
        iteration and counter, with a ragged particle count: trajectories equal
        the oracle's bit for bit."""
        cfg = cb.SimConfig(513, 600, init_counter=0xFFFFFF00, mode=mode)
        p = cb.init_particles(cfg)
        cb.brownian.run_steps(p, cfg, start_iteration=7)
        ref = oracle.brownian_init("philox", 513, 0xFFFFFF00)
        oracle.brownian_steps("philox", ref, 7, 600, init_ctr=0xFFFFFF00)
        for got, r in zip((p.x, p.y, p.vx, p.vy), ref):
            assert np.array_equal(host(got), r)

    def test_iteration_zero_rejected(self, cb):
        cfg = cb.SimConfig(4, 1)
        with pytest.raises(ValueError):
            cb.apply_forces_step(cb.init_particles(cfg), 0, cfg)

    def test_restart_matches_straight(self, cb, tmp_path):
        full = cb.run_sim(cb.SimConfig(300, 20))
        half = cb.run_sim(cb.SimConfig(300, 10, mode="per_step"))
        snap = tmp_path / "half.snap"
        cb.save_snapshot(snap, half.particles, next_iteration=11)
        particles, next_it = cb.load_snapshot(snap)
        resumed = cb.run_sim(cb.SimConfig(300, 10), particles=particles, start_iteration=next_it)
        assert resumed.checksum == full.checksum

    @pytest.mark.parametrize("explicit_pid", [False, True])
    def test_packed_records_match_host_layout(self, cb, oracle, explicit_pid):
        """cbrng_pack_records == numpy's `<Qdddd` records (brownian.py:209-223), and
        load_snapshot's device unpack inverts it."""
        import torch
        from paper_2310_19925_b200 import brownian

        cfg = cb.SimConfig(1003, 5, algorithm="squares")
        p = cb.run_sim(cfg, with_checksum=False).particles
        if explicit_pid:
            p = brownian.Particles(torch.arange(7, 7 + 3 * p.n, 3, device="cuda").to(torch.uint64),
                                   p.x, p.y, p.vx, p.vy)
        h = p.host()
        want = np.ascontiguousarray(np.column_stack(
            [h["pid"].astype("<u8")] + [h[k].astype("<f8").view("<u8") for k in ("x", "y", "vx", "vy")]))
        got = brownian._packed_records(p)
        assert got.tobytes() == want.tobytes()
        assert str(brownian.checksum(p)) == f"{oracle.fnv1a64(want.view(np.uint8).ravel()):016x}"

    def test_cfg3_full_size_spot_check(self, cb, oracle):
        """configs[2] at full size (10M particles x 10k steps, fused): particles are
        independent, so the oracle replays 24 pids spread over the range (both
        ends included) for all 10k steps and must match bit for bit."""
        n, steps = 10_000_000, 10_000
        cfg = cb.SimConfig(n, steps)
        p = cb.init_particles(cfg)
        cb.brownian.run_steps(p, cfg)
        rng = np.random.default_rng(3)
        pids = np.unique(np.concatenate([[0, 1, n // 2, n - 2, n - 1], rng.integers(0, n, 19)])).astype(np.uint64)
        ref = oracle.brownian_init("philox", pids.size, 0, pid=pids)
        oracle.brownian_steps("philox", ref, 1, steps, pid=pids)
        idx = pids.astype(np.int64)
        for got, r in zip((p.x, p.y, p.vx, p.vy), ref):
            assert np.array_equal(host(got)[idx], r)

    def test_checksum_rejects_unsorted_pids(self, cb):
        import torch
        from paper_2310_19925_b200 import brownian

        p = cb.init_particles(cb.SimConfig(64, 1))
        pid = torch.arange(64, device="cuda").to(torch.uint64)
        pid[40], pid[41] = 41, 40
        with pytest.raises(ValueError):
            brownian.checksum(brownian.Particles(pid, p.x, p.y, p.vx, p.vy))
        pid[40], pid[41] = 40, 40
        with pytest.raises(ValueError):
            brownian.checksum(brownian.Particles(pid, p.x, p.y, p.vx, p.vy))

    def test_shard_invariance_and_stats(self, cb):
        """pid-range shards (any count) reproduce the single run bit for bit."""
        import torch
        from paper_2310_19925_b200 import brownian, sharding

        cfg = cb.SimConfig(10_007, 50, algorithm="philox")
        whole = cb.run_sim(cfg, with_checksum=False).particles
        acc_whole = brownian.stats(whole)
        for world in (2, 3, 8):
            acc = torch.zeros(8, dtype=torch.int64, device="cuda")
            xs = []
            for r in range(world):
                lo, hi = sharding.shard_range(cfg.n_particles, r, world)
                p = brownian.init_particles(cfg, pid_base=lo, n=hi - lo)
                brownian.run_steps(p, cfg)
                brownian.stats(p, acc)
                xs.append(p.x)
            assert torch.equal(torch.cat(xs), whole.x)
            assert torch.equal(acc, acc_whole)


class TestSpotChecksAtScale:
    """BASELINE configs at full size, checked by size-independent properties:
    oracle spot checks at random positions and digest equality under sharding."""

    @pytest.mark.parametrize("alg", ["philox", "threefry", "squares"])
    def test_cfg2_uniform_f32_2p30_spot(self, cb, oracle, alg):
        n = 1 << 30
        out = cb.uniform_f32_array(cb.make_generator(alg, 42, 0), n)
        rng = np.random.default_rng(5)
        idx = np.concatenate([[0, 1, 2, 3, n - 4, n - 3, n - 2, n - 1], rng.integers(0, n // 4, 200) * 4])
        for i in idx:
            i = int(i) & ~3
            if alg == "squares":
                ref = oracle.words_to_f32(oracle.stream_words(alg, 42, 0, 4, block_ctr=i))
            else:
                ref = oracle.words_to_f32(oracle.stream_words(alg, 42, 0, 4, block_ctr=i // 4))
            assert np.array_equal(out[i:i + 4].cpu().numpy(), ref), i
        del out

    @pytest.mark.parametrize("alg", ["philox", "squares"])
    def test_fill_beyond_2p32_elements(self, cb, oracle, alg):
        """One f32 fill of 2^32 + 10 values (16 GiB; 64-bit unit indexing, and for
        Squares the 32-bit counter wrap inside the fill, bulk.py:268): spot checks
        around 2^32 and at both ends."""
        import torch

        n = (1 << 32) + 10
        out = cb.uniform_f32_array(cb.make_generator(alg, 7, 3), n)
        for i in (0, 4, (1 << 32) - 8, (1 << 32) - 4, 1 << 32, (1 << 32) + 4):
            bc = i if alg == "squares" else i // 4
            ref = oracle.words_to_f32(oracle.stream_words(alg, 7, 3, 4, block_ctr=bc & 0xFFFFFFFF))
            assert np.array_equal(out[i:i + 4].cpu().numpy(), ref), i
        ref = oracle.words_to_f32(oracle.stream_words(alg, 7, 3, 2, block_ctr=((n - 2) if alg == "squares" else (n - 2) // 4) & 0xFFFFFFFF,
                                                     lane=0 if alg == "squares" else (n - 2) % 4))
        assert np.array_equal(out[n - 2:].cpu().numpy(), ref)
        del out
        torch.cuda.empty_cache()

    def test_cfg5_multistream_sharded_digest(self, cb, oracle):
        """100M-stream layout, shortened to 4M streams x 256: digest of the
        whole == sum of shard digests; rows spot-checked against the oracle."""
        import torch
        from paper_2310_19925_b200 import bulk, sharding

        n, nw = 1 << 22, 256
        whole = bulk.prefix_words("philox", range(n), 0, nw)
        d_whole = sharding.digest_words(whole, 0)
        acc = torch.zeros(1, dtype=torch.int64, device="cuda")
        for r in range(4):
            lo, hi = sharding.shard_range(n, r, 4)
            part = bulk.prefix_words("philox", range(lo, hi), 0, nw)
            sharding.digest_words(part, lo * nw, acc)
        assert torch.equal(acc, d_whole)
        for row in (0, 1, n // 2, n - 1):
            assert np.array_equal(whole[row].cpu().numpy(), oracle.prefix_words_arange("philox", row, 1, 0, nw)[0])
        small = whole[:1000].cpu().numpy()
        assert sharding.digest_words_np(small.reshape(-1), 0) == int(
            sharding.digest_words(whole[:1000], 0).cpu().numpy()[0]) % 2**64


class TestApiSurface:
    """Reference API behaviours (generators.py:227-406, distributions.py) on the CUDA path."""

    @pytest.mark.parametrize("alg", ALGS)
    def test_copy_replays(self, cb, alg):
        g = cb.make_generator(alg, 123456789, 42)
        [g.next_u32() for _ in range(7)]
        h = g.copy()
        assert [g.next_u32() for _ in range(20)] == [h.next_u32() for _ in range(20)]
        assert np.array_equal(host(g.words(300)), host(h.words(300)))

    def test_generator_classes(self, cb, oracle):
        for cls, alg in ((cb.Philox, "philox"), (cb.Threefry, "threefry"), (cb.Squares, "squares"), (cb.Tyche, "tyche")):
            assert np.array_equal(host(cls(9, 2).words(77)), oracle.stream_words(alg, 9, 2, 77))

    def test_state_layout(self, cb):
        import struct

        g = cb.make_generator("threefry", 0x1122334455667788, 0x99AABBCC)
        [g.next_u32() for _ in range(6)]
        tag, seed, sc, ic, pos = struct.unpack("<BQIIB", g.state_bytes())
        assert (tag, seed, sc, ic, pos) == (1, 0x1122334455667788, 0x99AABBCC, 2, 2)

    def test_single_word_algorithms_reject_cache_pos(self, cb):
        import struct

        with pytest.raises(ValueError):
            cb.Generator.from_state_bytes(struct.pack("<BQIIB", 2, 1, 2, 3, 1))

    def test_squares_uses_low_32_seed_bits(self, cb):
        a = host(cb.make_generator("squares", 2**40 + 123, 0).words(64))
        b = host(cb.make_generator("squares", (2**40 + 123) & M32, 0).words(64))
        assert np.array_equal(a, b)

    def test_device_and_out_placement(self, cb, oracle):
        import torch

        ref = oracle.stream_words("philox", 5, 1, 1000)
        assert isinstance(cb.make_generator("philox", 5, 1).words(1000, device="cpu"), np.ndarray)
        out = torch.empty(1000, dtype=torch.uint32, device="cuda")
        assert cb.make_generator("philox", 5, 1).words(1000, out=out) is out
        assert np.array_equal(out.cpu().numpy(), ref)
        hout = np.empty(1000, np.uint32)
        cb.make_generator("philox", 5, 1).words(1000, out=hout)
        assert np.array_equal(hout, ref)
        pinned = torch.empty(1000, dtype=torch.uint32, pin_memory=True)
        cb.make_generator("philox", 5, 1).words(1000, out=pinned)
        assert np.array_equal(pinned.numpy(), ref)

    @pytest.mark.parametrize("alg", ["philox", "threefry", "squares", "tyche"])
    def test_normal2_resumed_mid_stream(self, cb, oracle, alg):
        g = cb.make_generator(alg, 8, 1)
        [g.next_u32() for _ in range(3)]
        z0, z1 = (host(z) for z in cb.normal2_array(g, 1001))
        r0, r1 = oracle.words_to_normal2(oracle.stream_words(alg, 8, 1, 3 + 4 * 1001)[3:])
        for got, r in ((z0, r0), (z1, r1)):
            assert np.all(np.abs(got - r) <= BM_ULP * np.spacing(np.maximum(np.abs(r), 1.0)))
        assert g._block_ctr == (1 + 1001 if alg in ("philox", "threefry") else 3 + 4 * 1001)

    def test_draw_accounting(self, cb, oracle):
        g = cb.make_generator("threefry", 8, 8)
        w = oracle.stream_words("threefry", 8, 8, 16)
        cb.uniform_f64(g); cb.uniform_f32(g); cb.draw_double2(g); cb.range_u32(g, 17); cb.normal2(g)
        assert g.next_u32() == int(w[12])

    def test_prefix_words_device_inputs(self, cb, oracle, golden_arrays):
        import torch
        from paper_2310_19925_b200 import bulk

        seeds = torch.from_numpy(golden_arrays["prefix_seeds"]).cuda()
        ctrs = torch.from_numpy(golden_arrays["prefix_ctrs"]).cuda()
        got = bulk.prefix_words("threefry", seeds, ctrs, 19)
        assert got.is_cuda
        assert np.array_equal(got.cpu().numpy(), golden_arrays["prefix_threefry_19"])

    def test_tyche_fill_c_abi(self, cb, oracle):
        """_kernels.tyche_fill drop-in: state updated in place (synchronous)."""
        import ctypes

        import torch
        from paper_2310_19925_b200 import _lib

        st = np.array(oracle.tyche_init(77, 3), dtype=np.uint64)
        out = torch.empty(1000, dtype=torch.uint32, device="cuda")
        _lib.check(_lib.lib().cbrng_tyche_fill(st.ctypes.data, 1000, out.data_ptr(), None))
        words, final = oracle.stream_words("tyche", 77, 3, 1000, tyche_state=oracle.tyche_init(77, 3))
        assert np.array_equal(out.cpu().numpy(), words)
        assert tuple(int(v) for v in st) == final


class TestShardingAndKernelsModule:
    def test_uniform_f32_shards_concatenate(self, cb, oracle):
        import torch
        from paper_2310_19925_b200 import sharding

        n = (1 << 20) + 6
        whole = cb.uniform_f32_array(cb.make_generator("threefry", 42, 3), n)
        for world in (1, 2, 3, 8):
            parts = [sharding.uniform_f32_shard("threefry", 42, 3, n, r, world)[2] for r in range(world)]
            assert torch.equal(torch.cat(parts), whole)

    def test_run_sim_shard_stats_invariant(self, cb):
        import torch
        from paper_2310_19925_b200 import sharding

        cfg = cb.SimConfig(5003, 30)
        accs = []
        for world in (1, 4):
            acc = torch.zeros(8, dtype=torch.int64, device="cuda")
            for r in range(world):
                _, a = sharding.run_sim_shard(cfg, r, world)  # no process group: local sums
                acc += a
            accs.append(acc)
        assert torch.equal(accs[0], accs[1])

    def test_kernels_module_drop_in(self, cb, oracle):
        from paper_2310_19925_b200 import _kernels

        st = np.array(oracle.tyche_init(77, 3), dtype=np.uint64)
        out = np.empty(333, np.uint32)
        _kernels.tyche_fill(st, out)
        words, final = oracle.stream_words("tyche", 77, 3, 333, tyche_state=oracle.tyche_init(77, 3))
        assert np.array_equal(out, words) and tuple(int(v) for v in st) == final
        seeds = np.arange(10, 20, dtype=np.uint64)
        scs = np.full(10, 4, np.uint64)
        blk = np.empty((10, 4), np.uint32)
        _kernels.philox_block_lanes(seeds, scs, 1, blk)
        assert np.array_equal(blk, oracle.prefix_words("philox", seeds, 4, 8)[:, 4:8])
        assert _kernels.fnv1a64(np.zeros(40, np.uint8)) == oracle.fnv1a64(bytes(40))


class TestMicroBenchmark:
    """The reference's harness-shape tests (pkg/tests/test_bench.py); timings are not asserted."""

    def test_rows(self, cb):
        rows = cb.micro_benchmark("philox", [1, 10, 100], repetitions=2)
        assert [r.length for r in rows] == [1, 10, 100]
        assert all(r.median_ns > 0 and r.words_per_second > 0 and r.algorithm == "philox" for r in rows)

    def test_amortizes(self, cb):
        rows = cb.micro_benchmark("squares", [1, 1_000_000], repetitions=3)
        assert rows[1].median_ns / rows[1].length < rows[0].median_ns / rows[0].length


class TestHostPipelinedFills:
    """Large fills into host memory stream chunk by chunk (pipelined D2H); the
    values and the generator state must equal the one-shot device fill."""

    @pytest.mark.parametrize("alg", ["philox", "threefry", "squares"])
    def test_uniform_f32_to_pinned_host(self, cb, alg):
        import torch

        n = (1 << 25) + 12345
        g_host, g_dev = cb.make_generator(alg, 77, 5), cb.make_generator(alg, 77, 5)
        for g in (g_host, g_dev):
            g.next_u32(); g.next_u32(); g.next_u32()  # start mid-block
        out = torch.empty(n, dtype=torch.float32, pin_memory=True)
        got = cb.uniform_f32_array(g_host, n, out=out)
        assert got is out
        ref = host(cb.uniform_f32_array(g_dev, n))
        assert np.array_equal(out.numpy(), ref)
        assert g_host.state_bytes() == g_dev.state_bytes()
        assert g_host.next_u32() == g_dev.next_u32()

    def test_normal2_and_words_to_cpu(self, cb):
        n = (1 << 24) + 7
        a = cb.normal2_array(cb.make_generator("philox", 3, 1), n, device="cpu")
        b = cb.normal2_array(cb.make_generator("philox", 3, 1), n)
        assert all(isinstance(x, np.ndarray) for x in a)
        assert np.array_equal(a[0], host(b[0])) and np.array_equal(a[1], host(b[1]))
        w = cb.make_generator("squares", 9, 2).words((1 << 26) + 1, device="cpu")
        assert np.array_equal(w, host(cb.make_generator("squares", 9, 2).words((1 << 26) + 1)))

    def test_prefix_uniform_f32_to_pinned_host(self, cb):
        import torch

        from paper_2310_19925_b200 import bulk

        n, nw = (1 << 17) + 3, 256
        out = torch.empty(n * nw, dtype=torch.float32, pin_memory=True)
        bulk.prefix_uniform_f32("tyche", range(11, 11 + n), 4, nw, out=out)
        ref = host(bulk.prefix_uniform_f32("tyche", range(11, 11 + n), 4, nw)).reshape(-1)
        assert np.array_equal(out.numpy(), ref)
        seeds = np.arange(5, 5 + n, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        got = bulk.prefix_uniform_f32("philox", seeds, 0, nw, device="cpu")
        assert isinstance(got, np.ndarray) and got.shape == (n, nw)
        assert np.array_equal(got, host(bulk.prefix_uniform_f32("philox", seeds, 0, nw)))


class TestReentrancy:
    """The C ABI is reentrant (no global mutable state but thread-safe launch
    caches; thread-local error text), as the reference's nogil numba kernels are
    called from a thread pool (brownian.py:185-191): concurrent calls from
    several host threads, each on its own CUDA stream, give the sequential results."""

    def test_concurrent_fills_and_errors(self, cb, oracle):
        import threading

        import torch

        from paper_2310_19925_b200 import _lib

        lib = _lib.lib()
        n = 1 << 20
        jobs = [(a, s) for a in range(3) for s in range(4)]
        outs = {j: torch.empty(n, dtype=torch.uint32, device="cuda") for j in jobs}
        errs = {}

        def work(j):
            a, s = j
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                rc = lib.cbrng_words(a, 1000 + s, s, 0, None, n, outs[j].data_ptr(), None, int(st.cuda_stream))
                bad = lib.cbrng_words(9, 0, 0, 0, None, 1, outs[j].data_ptr(), None, int(st.cuda_stream))
                errs[j] = (rc, bad, lib.cbrng_last_error().decode())
            st.synchronize()

        threads = [threading.Thread(target=work, args=(j,)) for j in jobs]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        names = ["philox", "threefry", "squares"]
        for (a, s), (rc, bad, msg) in errs.items():
            assert rc == 0 and bad == _lib.CBRNG_EALG and "algorithm" in msg
            assert np.array_equal(host(outs[(a, s)]), oracle.stream_words(names[a], 1000 + s, s, n))
