"""Generate the committed golden fixtures by running the REFERENCE package.

Test infrastructure only. Imports the upstream `cbrng` package from
/root/reference/pkg/src (available in the build container, absent on the GPU
box) and freezes its outputs into tests/golden/golden.json (+ golden.npz), so
the oracle and the CUDA path can be checked against the reference itself
without the reference being present at run time.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every value below is computed by a reference call named next to it (file:line
in /root/reference/pkg/src/cbrng).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import cbrng  # noqa: E402  (reference package)
from cbrng import bulk, distributions, brownian  # noqa: E402
from cbrng.generators import (  # noqa: E402
    Algorithm, Generator, make_generator, philox_block, threefry_block,
    squares_key, squares_round, tyche_init, tyche_next,
)

OUT = Path(__file__).resolve().parent
M32 = 0xFFFFFFFF
ALGS = ["philox", "threefry", "squares", "tyche"]


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    g: dict = {"generator": "tests/golden/make_golden.py", "reference": "cbrng 0.1.0 (/root/reference/pkg/src)"}
    arrays: dict[str, np.ndarray] = {}

    # --- block-function KATs (inputs from reference tests/test_generators.py:33-68)
    philox_in = [((0, 0, 0, 0), (0, 0)), ((M32,) * 4, (M32, M32)),
                 ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0))]
    g["philox_kat"] = [[list(c), list(k), list(philox_block(k, c))] for c, k in philox_in]  # generators.py:101
    tf_in = [((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
              (0xA4093822, 0x299F31D0, 0x082EFA98, 0xEC4E6C89)),
             ((0, 0, 0, 0), (0, 0, 0, 0)), ((M32,) * 4, (M32,) * 4)]
    g["threefry_kat_20"] = [[list(c), list(k), list(threefry_block(k, c))] for c, k in tf_in]  # :125
    g["threefry_kat_13"] = [[[0] * 4, [0] * 4, list(threefry_block((0,) * 4, (0,) * 4, rounds=13))]]
    g["squares_kat"] = [[s, squares_key(s), [squares_round(squares_key(s), c) for c in range(3)]]
                        for s in (0, 1, 0xDEADBEEF)]  # :157, :173
    st = tyche_init(0x1234, 0)  # :204
    words = []
    for _ in range(4):
        w, st = tyche_next(st)
        words.append(w)
    g["tyche_kat"] = {"seed": 0x1234, "ctr": 0, "state": list(tyche_init(0x1234, 0)), "words": words}

    # random block inputs -> outputs (vector cipher parity, bulk.py:49, :69, :95)
    rng = np.random.default_rng(11)
    c = rng.integers(0, 2**32, (4, 256), dtype=np.uint32)
    k = rng.integers(0, 2**32, (4, 256), dtype=np.uint32)
    arrays["blk_ctr"] = c
    arrays["blk_key"] = k
    arrays["blk_philox"] = np.stack(bulk.philox4x32(*c, k[0], k[1]))
    arrays["blk_threefry"] = np.stack(bulk.threefry4x32(*c, *k))
    sq_ctr = rng.integers(0, 2**63, 256, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 256).astype(np.uint64)
    sq_key = rng.integers(0, 2**63, 256, dtype=np.uint64) | np.uint64(1)
    arrays["blk_sq_ctr"] = sq_ctr
    arrays["blk_sq_key"] = sq_key
    arrays["blk_squares"] = bulk.squares32(sq_ctr, sq_key)
    arrays["blk_sq_seeds"] = rng.integers(0, 2**64, 256, dtype=np.uint64)
    arrays["blk_sq_keys_of_seeds"] = bulk.squares_keys(arrays["blk_sq_seeds"])
    arrays["blk_tyche_state"] = np.stack(bulk.tyche_mix(*c))

    # --- stream prefixes at (42, 0) (test_generators.py:72-81)
    g["stream_seed42"] = {a: [int(w) for w in make_generator(a, 42, 0).words(8)] for a in ALGS}

    # --- cfg1: Philox u32 fill 2^20, seed 42, ctr 0 (BASELINE.json configs[0])
    w = make_generator("philox", 42, 0).words(2**20)  # generators.py:322 -> bulk.py:223
    g["cfg1"] = {"n": 2**20, "sha256": sha(w), "sha16": sha16(w), "first": int(w[0]), "last": int(w[-1])}

    # --- single-stream words for several (seed, ctr) pairs, full digests + stored prefixes
    pairs = [(42, 0), (0xFEEDFACE, 3), (2**64 - 1, M32), (0x123456789ABCDEF0, 7)]
    g["stream_pairs"] = [[s, c_] for s, c_ in pairs]
    g["stream_digests"] = {}
    for a in ALGS:
        g["stream_digests"][a] = []
        for i, (s, c_) in enumerate(pairs):
            w = make_generator(a, s, c_).words(65536 + 3)
            g["stream_digests"][a].append(sha(w))
            arrays[f"stream_{a}_{i}"] = w[:1027]

    # block-counter wrap (generators.py:288, bulk.py:215-217): start 3 blocks before 2^32
    g["wrap"] = {}
    for a in ALGS:
        gen = make_generator(a, 5, 6)
        gen._block_ctr = 2**32 - 3
        w = gen.words(200)
        arrays[f"wrap_{a}"] = w
        g["wrap"][a] = {"block_ctr_after": gen._block_ctr, "cache_pos_after": gen._cache_pos}

    # engine state after mixed scalar/bulk use (bulk.py:242-266; generators.py:345-353)
    g["state_after"] = {}
    for a in ALGS:
        gen = make_generator(a, 0xFEEDFACE, 3)
        seq = [gen.next_u32() for _ in range(3)]
        seq += [int(x) for x in gen.words(130)]
        seq += [gen.next_u32() for _ in range(2)]
        seq += [int(x) for x in gen.words(1001)]
        g["state_after"][a] = {"state_bytes": gen.state_bytes().hex(), "n": len(seq), "sha": sha(np.array(seq, dtype=np.uint32)),
                               "tyche_state": list(gen._tyche_state) if gen._tyche_state else None}

    # restore mid-block (generators.py:355-374, test_acceptance.py:64-72)
    g["restore_split"] = 3731

    # --- distributions (distributions.py:99-120)
    g["uniform_f32_2p20"] = {a: sha(distributions.uniform_f32_array(make_generator(a, 42, 0), 2**20)) for a in ALGS}
    g["uniform_f64_2p19"] = {a: sha(distributions.uniform_f64_array(make_generator(a, 42, 0), 2**19)) for a in ALGS}
    for a in ALGS:
        arrays[f"uf32_{a}"] = distributions.uniform_f32_array(make_generator(a, 99, 2), 1029)
        arrays[f"uf64_{a}"] = distributions.uniform_f64_array(make_generator(a, 99, 2), 1029)
        z0, z1 = distributions.normal2_array(make_generator(a, 42, 0), 4099)
        arrays[f"n2bulk_{a}_z0"], arrays[f"n2bulk_{a}_z1"] = z0, z1
        gen = make_generator(a, 42, 0)
        sc = np.array([distributions.normal2(gen) for _ in range(4099)])  # scalar libm path :72-81
        arrays[f"n2scalar_{a}"] = sc
    z0, z1 = distributions.normal2_array(make_generator("philox", 42, 0), 2**19)
    g["normal2_2p19_philox"] = {"z0_sha16": sha16(z0), "z1_sha16": sha16(z1), "z0_0": float(z0[0])}

    # --- multi-stream prefix words (bulk.py:162-207)
    g["prefix_arange_2p16_256"] = {a: sha(bulk.prefix_words(Algorithm.from_name(a), np.arange(2**16, dtype=np.uint64), 0, 256)) for a in ALGS}
    rng = np.random.default_rng(15)
    seeds = rng.integers(0, 2**64, size=64, dtype=np.uint64)
    ctrs = rng.integers(0, 2**32, size=64, dtype=np.uint32)
    arrays["prefix_seeds"] = seeds
    arrays["prefix_ctrs"] = ctrs
    for a in ALGS:
        for nw in (1, 4, 7, 19):
            arrays[f"prefix_{a}_{nw}"] = bulk.prefix_words(Algorithm.from_name(a), seeds, ctrs, nw)
        arrays[f"prefix_{a}_scalarctr"] = bulk.prefix_words(Algorithm.from_name(a), seeds, np.uint32(9), 12)

    # --- Brownian (brownian.py:112-195)
    g["brownian_1000x100"] = {a: str(brownian.run_sim(brownian.SimConfig(1000, 100, threads=1, algorithm=a)).checksum) for a in ALGS}
    g["brownian_1e5x1e3_philox"] = str(brownian.run_sim(brownian.SimConfig(100_000, 1000, threads=8)).checksum)
    cases = {
        "default": dict(n_particles=97, steps=13),
        "drag": dict(n_particles=64, steps=7, gamma=0.5, mass=2.0, dt=0.02, init_counter=5),
        "nodt": dict(n_particles=16, steps=3, dt=0.0),
    }
    g["brownian_cases"] = {}
    for name, kw in cases.items():
        for a in ALGS:
            cfg = brownian.SimConfig(algorithm=a, **kw)
            p0 = brownian.init_particles(cfg)
            r = brownian.run_sim(cfg)
            for f in ("x", "y", "vx", "vy"):
                arrays[f"bw_{name}_{a}_init_{f}"] = getattr(p0, f)
                arrays[f"bw_{name}_{a}_{f}"] = getattr(r.particles, f)
            g["brownian_cases"][f"{name}_{a}"] = {"cfg": {**kw, "algorithm": a}, "checksum": str(r.checksum)}

    # --- FNV-1a 64 (_kernels.py:89-96)
    from cbrng import _kernels
    blob = np.frombuffer(bytes(range(256)) * 3, dtype=np.uint8).copy()
    g["fnv"] = {"empty": _kernels.FNV_OFFSET_BASIS, "zero40": int(_kernels.fnv1a64(np.zeros(40, np.uint8))),
                "bytes0_255x3": int(_kernels.fnv1a64(blob))}

    # --- cross-process determinism panel (tests/_digest_runner.py)
    sys.path.insert(0, "/root/reference/pkg/tests")
    import _digest_runner
    g["panel"] = {"pairs": [[s, c_] for s, c_ in _digest_runner.stream_panel()], "words": _digest_runner.WORDS,
                  "sha256": _digest_runner.panel_digest()}

    # --- statistical battery (stats.py): SURVEY §8(f) rank 1
    from cbrng import stats as st
    g["battery_16MiB"] = {}
    for a in ALGS:
        reps = st.run_battery(Algorithm.from_name(a), 16 * 2**20)
        g["battery_16MiB"][a] = [st.report_to_dict(r) for r in reps]
    blob = make_generator("squares", 3, 1).words(100_003).astype("<u4").tobytes()[:400_010]
    g["blob_tests"] = {"monobit": st.report_to_dict(st.monobit(blob)),
                       "chi_square_bytes": st.report_to_dict(st.chi_square_bytes(blob)),
                       "ks_uniform": st.report_to_dict(st.ks_uniform(distributions.words_to_unit_doubles(
                           make_generator("threefry", 5, 0).words(20_000))))}
    g["avalanche_20000"] = {}
    for a in ALGS:
        av = st.avalanche_stats(Algorithm.from_name(a), 20_000)
        g["avalanche_20000"][a] = {"mean": av.mean_hamming, "rates": av.bit_flip_rates.tolist(), "z": av.z}
    spec = st.InterleaveSpec(n_streams=1000, draws_per_stream=3, iterations=4)
    g["interleave_1000x3x4"] = {a: sha(np.frombuffer(st.interleave_stream(spec, Algorithm.from_name(a), 77),
                                                     dtype=np.uint8)) for a in ALGS}

    (OUT / "golden.json").write_text(json.dumps(g, indent=1, sort_keys=True) + "\n")
    np.savez_compressed(OUT / "golden.npz", **arrays)
    print("wrote", OUT / "golden.json", OUT / "golden.npz",
          sum(v.nbytes for v in arrays.values()), "array bytes")


if __name__ == "__main__":
    main()
