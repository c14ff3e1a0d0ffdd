"""Time the REFERENCE package itself (numpy/numba, installed into baseline/_ref) on
bounded samples of each BASELINE config, on this host's cores.

    PYTHONPATH=baseline/_ref python tools/ref_package_bench.py [--quick]

bench.py runs this in a subprocess (when baseline/_ref exists) and reports the
numbers next to the C port's (`cpu_baseline.reference_package`). Prints one JSON
object. Each measurement runs the call once untimed first (numba compiles on
first use) and then times `reps` calls. Reference entry points:
  configs[1]  distributions.uniform_f32_array (distributions.py:105-107) x 3
              generators + bulk.prefix_words('tyche', ..., 256) (bulk.py:162-207)
  configs[2]  brownian.run_sim(SimConfig(n, steps, threads=nproc)) (brownian.py:164-195)
  configs[3]  distributions.normal2_array (distributions.py:110-120)
  configs[4]  bulk.prefix_words('philox', arange(n), 0, 256) (bulk.py:162-207)
"""

from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")

import numpy as np  # noqa: E402


def timed(fn, reps=1):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps


def main() -> None:
    quick = "--quick" in sys.argv
    import cbrng
    from cbrng import brownian, bulk, distributions
    from cbrng.generators import Algorithm, make_generator

    nproc = os.cpu_count() or 1
    out = {"package": getattr(cbrng, "__file__", "?"), "threads_available": nproc}
    n1 = 1 << (20 if quick else 22)
    rows = n1 // 256

    def cfg1():
        for a in ("philox", "threefry", "squares"):
            distributions.uniform_f32_array(make_generator(a, 42, 0), n1)
        w = bulk.prefix_words(Algorithm.TYCHE, np.arange(rows, dtype=np.uint64), 0, 256)
        ((w >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24))

    t = timed(cfg1)
    out["configs[1]"] = {"value": 4 * n1 / t / 1e9, "unit": "Gsamples/s", "cores": 1,
                         "sample": f"uniform_f32_array x3 (2^{n1.bit_length() - 1}) + tyche prefix_words "
                                   f"({rows} x 256)", "seconds": t}
    n2, s2 = (100_000, 10) if quick else (1_000_000, 10)
    t = timed(lambda: brownian.run_sim(brownian.SimConfig(n2, s2, threads=nproc)))
    out["configs[2]"] = {"value": n2 * s2 / t, "unit": "particle-steps/s", "cores": nproc,
                         "sample": f"run_sim(SimConfig({n2}, {s2}, threads={nproc})) wall incl. init",
                         "seconds": t}
    n3 = 1 << (18 if quick else 21)
    t = timed(lambda: distributions.normal2_array(make_generator("philox", 42, 0), n3))
    out["configs[3]"] = {"value": 2 * n3 / t / 1e9, "unit": "Gvalues/s", "cores": 1,
                         "sample": f"normal2_array(philox, 2^{n3.bit_length() - 1} pairs)", "seconds": t}
    n4 = 100_000 if quick else 1_000_000
    t = timed(lambda: bulk.prefix_words(Algorithm.PHILOX, np.arange(n4, dtype=np.uint64), 0, 256))
    out["configs[4]"] = {"value": n4 * 256 / t / 1e9, "unit": "Gwords/s", "cores": 1,
                         "sample": f"prefix_words(philox, arange({n4}), 0, 256)", "seconds": t}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
