"""Scalar (per-call) API latency: this package vs the reference package, same host.

    python tools/bench_scalar.py                       # both (reference from baseline/_ref)
    python tools/bench_scalar.py --impl b200|reference # one, prints one JSON object

The reference's scalar path is pure Python over ints (generators.py:101-224,
295-320; distributions.py:42-81); ours serves scalar draws from a prefetched
window of GPU-generated words and evaluates the scalar block functions as
one-lane kernels. Timed per call with perf_counter_ns, median of repetitions:
  next_u32 x L after construction (L = 1, 10, 100, 1000)  generators.py:295-320
  normal2(g) x 1000                                       distributions.py:72-81
  philox_block / threefry_block / squares_round / tyche_init, per call
  micro_benchmark(L = 1, 10, 100, 10^4, 10^6)             bench.py:31-53
"""

from __future__ import annotations

import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def med_ns(fn, reps: int) -> float:
    fn()
    s = []
    for _ in range(reps):
        t = time.perf_counter_ns()
        fn()
        s.append(time.perf_counter_ns() - t)
    return statistics.median(s)


def run(impl: str) -> dict:
    if impl == "b200":
        sys.path.insert(0, str(ROOT))
        import paper_2310_19925_b200 as cb
        from paper_2310_19925_b200 import microbench as mb
    else:
        import cbrng as cb
        from cbrng import bench as mb
    out = {"impl": impl, "package": cb.__file__}
    for alg in ("philox", "threefry", "squares", "tyche"):
        row = {}
        for L in (1, 10, 100, 1000):
            def draw(L=L):
                g = cb.make_generator(alg, 7, 3)
                for _ in range(L):
                    g.next_u32()
            row[f"construct+next_u32x{L}_us"] = round(med_ns(draw, 5 if L >= 1000 else 20) / 1e3, 2)

        def n2():
            g = cb.make_generator(alg, 7, 3)
            for _ in range(1000):
                cb.normal2(g)
        row["normal2x1000_us_per_call"] = round(med_ns(n2, 3) / 1e3 / 1000, 3)
        rows = mb.micro_benchmark(alg, [1, 10, 100, 10_000, 1_000_000], repetitions=5)
        row["micro_benchmark"] = {r.length: {"median_ns": r.median_ns, "words_per_second": r.words_per_second}
                                  for r in rows}
        out[alg] = row
    blk = {}
    blk["philox_block_us"] = round(med_ns(lambda: cb.philox_block((1, 2), (3, 4, 5, 6)), 50) / 1e3, 2)
    blk["threefry_block_us"] = round(med_ns(lambda: cb.threefry_block((1, 2, 3, 4), (5, 6, 7, 8)), 50) / 1e3, 2)
    k = cb.squares_key(7)
    blk["squares_round_us"] = round(med_ns(lambda: cb.squares_round(k, 12345), 50) / 1e3, 2)
    blk["tyche_init_us"] = round(med_ns(lambda: cb.tyche_init(7, 3), 50) / 1e3, 2)
    out["block_functions"] = blk
    return out


def main() -> None:
    if "--impl" in sys.argv:
        print(json.dumps(run(sys.argv[sys.argv.index("--impl") + 1])), flush=True)
        return
    res = {"b200": run("b200")}
    ref = ROOT / "baseline" / "_ref"
    if (ref / "cbrng").exists():
        env = dict(os.environ, PYTHONPATH=str(ref), NUMBA_CACHE_DIR="/tmp/numba_cache_ref")
        r = subprocess.run([sys.executable, __file__, "--impl", "reference"], env=env, capture_output=True,
                           text=True, timeout=1200)
        res["reference"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {
            "error": r.stderr[-500:]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
