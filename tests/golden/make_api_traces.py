"""Freeze random API-call traces of the REFERENCE package into
tests/golden/api_traces.json (test infrastructure only).

Each trace builds a reference Generator and applies a random sequence of the
drop-in API's calls — scalar draws (generators.py:295-320, distributions.py:
42-81), bulk draws (words / uniform_*_array / normal2_array / fill_bytes,
generators.py:322-330, distributions.py:84-120), copy and state_bytes round
trips (generators.py:332-374) — recording every result and the 18-byte state
after every call. tests/test_gpu_api_traces.py replays the same sequences
through paper_2310_19925_b200 on the GPU: integer results, exact float maps and
states must match bit for bit, Box-Muller values within the 4-ulp tolerance.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_api_traces.py
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import struct
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from cbrng import distributions as D  # noqa: E402  (reference package)
from cbrng.generators import Generator, make_generator  # noqa: E402

OUT = Path(__file__).resolve().parent / "api_traces.json"
ALGS = ["philox", "threefry", "squares", "tyche"]
OPS = ["next_u32", "next_u64", "words", "uniform_f32", "uniform_f64", "uniform_f32_array", "uniform_f64_array",
       "normal2", "normal2_array", "range_u32", "fill_bytes", "draw_double2", "copy", "restore"]


def h16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def f64bits(x: float) -> str:
    return struct.pack("<d", float(x)).hex()


def apply(g: Generator, op: str, arg: int):
    """Run one op on the reference generator; returns (new generator, JSON-able result)."""
    if op == "next_u32":
        return g, g.next_u32()
    if op == "next_u64":
        return g, g.next_u64()
    if op == "words":
        w = np.asarray(g.words(arg), np.uint32)
        return g, {"sha": h16(w.tobytes()), "head": [int(x) for x in w[:3]]}
    if op == "uniform_f32":
        return g, np.float32(D.uniform_f32(g)).tobytes().hex()
    if op == "uniform_f64":
        return g, f64bits(D.uniform_f64(g))
    if op == "uniform_f32_array":
        return g, h16(np.asarray(D.uniform_f32_array(g, arg), np.float32).tobytes())
    if op == "uniform_f64_array":
        return g, h16(np.asarray(D.uniform_f64_array(g, arg), np.float64).tobytes())
    if op == "normal2":
        z0, z1 = D.normal2(g)
        return g, [float(z0), float(z1)]
    if op == "normal2_array":
        z0, z1 = D.normal2_array(g, arg)
        return g, [[float(v) for v in z0], [float(v) for v in z1]]
    if op == "range_u32":
        return g, D.range_u32(g, arg)
    if op == "fill_bytes":
        return g, D.fill_bytes(g, arg).hex()
    if op == "draw_double2":
        d = D.draw_double2(g)
        return g, [f64bits(d.x), f64bits(d.y)]
    if op == "copy":
        return g.copy(), None
    if op == "restore":
        return Generator.from_state_bytes(g.state_bytes()), None
    raise ValueError(op)


def bulk_traces(rnd: random.Random) -> list:
    """Random calls of the multi-stream and vector entry points (bulk.py:49-296)."""
    from cbrng import bulk
    from cbrng.generators import Algorithm

    out = []
    rng = np.random.default_rng(19925)
    for t in range(48):
        alg = ALGS[t % 4]
        a = Algorithm.from_name(alg)
        n = rnd.choice([1, 2, 31, 32, 33, 257, 1000])
        nw = rnd.choice([1, 3, 4, 8, 16, 17, 36, 256])
        seeds = rng.integers(0, 2**64, size=n, dtype=np.uint64)
        ctrs = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        scalar_ctr = rnd.random() < 0.5
        c_arg = int(ctrs[0]) if scalar_ctr else ctrs
        w = bulk.prefix_words(a, seeds, c_arg, nw)
        out.append({"call": "prefix_words", "alg": alg, "seeds": [int(x) for x in seeds],
                    "ctrs": int(ctrs[0]) if scalar_ctr else [int(x) for x in ctrs], "nwords": nw,
                    "sha": h16(np.ascontiguousarray(w, np.uint32).tobytes())})
        f = bulk.first_words(a, seeds, c_arg)
        out.append({"call": "first_words", "alg": alg, "seeds": [int(x) for x in seeds],
                    "ctrs": int(ctrs[0]) if scalar_ctr else [int(x) for x in ctrs],
                    "sha": h16(np.ascontiguousarray(f, np.uint32).tobytes())})
        src = bulk.AlgorithmSource(a)
        seed, ctr, m = int(seeds[0]), int(ctrs[0]), rnd.choice([1, 5, 129, 5000])
        out.append({"call": "source_stream_words", "alg": alg, "seed": seed, "ctr": ctr, "n": m,
                    "sha": h16(np.ascontiguousarray(src.stream_words(seed, ctr, m), np.uint32).tobytes())})
    v = {k: rng.integers(0, 2**32, size=777, dtype=np.uint64).astype(np.uint32) for k in "abcdefgh"}
    out.append({"call": "philox4x32", "in": {k: [int(x) for x in v[k]] for k in "abcdef"},
                "sha": h16(np.stack(bulk.philox4x32(v["a"], v["b"], v["c"], v["d"], v["e"], v["f"])).astype(np.uint32).tobytes())})
    out.append({"call": "threefry4x32", "in": {k: [int(x) for x in v[k]] for k in "abcdefgh"},
                "sha": h16(np.stack(bulk.threefry4x32(*(v[k] for k in "abcdefgh"))).astype(np.uint32).tobytes())})
    s64 = rng.integers(0, 2**64, size=777, dtype=np.uint64)
    keys = bulk.squares_keys(s64)
    out.append({"call": "squares_keys", "seeds": [int(x) for x in s64], "sha": h16(np.asarray(keys, np.uint64).tobytes())})
    c64 = rng.integers(0, 2**64, size=777, dtype=np.uint64)
    out.append({"call": "squares32", "ctr": [int(x) for x in c64], "key": [int(x) for x in keys],
                "sha": h16(np.asarray(bulk.squares32(c64, keys), np.uint32).tobytes())})
    ti = bulk.tyche_init(s64, v["a"])
    out.append({"call": "tyche_init", "seeds": [int(x) for x in s64], "ctrs": [int(x) for x in v["a"]],
                "sha": h16(np.stack(ti).astype(np.uint32).tobytes())})
    tm = bulk.tyche_mix(v["a"], v["b"], v["c"], v["d"])
    out.append({"call": "tyche_mix", "in": {k: [int(x) for x in v[k]] for k in "abcd"},
                "sha": h16(np.stack(tm).astype(np.uint32).tobytes())})
    for steps in (0, 1, 7, 1000):
        st = (int(v["a"][0]), int(v["b"][0]), int(v["c"][0]), int(v["d"][0]))
        out.append({"call": "tyche_advance_state", "state": list(st), "steps": steps,
                    "res": [int(x) for x in bulk.tyche_advance_state(st, steps)]})
    return out


def main() -> None:
    rnd = random.Random(2310_19925)
    traces = []
    for alg in ALGS:
        for t in range(24):
            seed = rnd.choice([0, 42, 0xDEADBEEF, rnd.getrandbits(64)])
            ctr = rnd.choice([0, 1, 0xFFFFFFFF, rnd.getrandbits(32)])
            g = make_generator(alg, seed, ctr)
            steps = []
            for _ in range(rnd.randint(6, 16)):
                op = rnd.choice(OPS)
                arg = 0
                if op in ("words", "uniform_f32_array", "uniform_f64_array"):
                    arg = rnd.choice([0, 1, 2, 3, 5, 127, 128, 129, 1000, 4099, rnd.randint(1, 70000)])
                elif op == "normal2_array":
                    arg = rnd.choice([0, 1, 3, 17])
                elif op == "range_u32":
                    arg = rnd.choice([1, 2, 6, 1000, 0xFFFFFFFF, rnd.randint(1, 0xFFFFFFFF)])
                elif op == "fill_bytes":
                    arg = rnd.choice([0, 1, 3, 4, 5, 33])
                g, res = apply(g, op, arg)
                steps.append({"op": op, "arg": arg, "res": res, "state": g.state_bytes().hex()})
            traces.append({"alg": alg, "seed": seed, "ctr": ctr, "steps": steps})
    OUT.write_text(json.dumps({"generator": "tests/golden/make_api_traces.py",
                               "reference": "cbrng 0.1.0 (/root/reference/pkg/src)", "traces": traces,
                               "bulk": bulk_traces(rnd)}, indent=0))
    print("wrote", OUT, sum(len(t["steps"]) for t in traces), "steps")


if __name__ == "__main__":
    main()
