"""Throughput of the fused battery producers on one GPU."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19925_b200 import stats as st  # noqa: E402


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {}
n = 1 << 28
for alg in ("philox", "threefry", "squares"):
    t = timed(lambda a=alg: st.histogram_stream(a, 1, 0, n))
    res[f"stream_hist_{alg}_GBps_tested"] = round(4 * n / t / 1e9, 1)
spec = st.InterleaveSpec(n_streams=16_000, draws_per_stream=3, iterations=1000)
for alg in ("philox", "tyche"):
    t = timed(lambda a=alg: st.interleave_histogram(spec, a, 7), reps=1)
    res[f"interleave_hist_{alg}_GBps_tested"] = round(spec.total_bytes / t / 1e9, 2)
t = timed(lambda: st.avalanche_stats("philox", 1_000_000), reps=1)
res["avalanche_1e6_s"] = round(t, 4)
for alg in ("philox", "tyche"):
    t0 = time.perf_counter()
    st.run_battery(alg, 16 * 2**20)
    res[f"run_battery_16MiB_{alg}_s"] = round(time.perf_counter() - t0, 3)

# §8(f) rank 2: raw emission to /dev/null (PCIe D2H + host write bound)
from paper_2310_19925_b200 import emit, make_generator  # noqa: E402

with open("/dev/null", "wb") as sink:
    emit.emit_words(make_generator("philox", 1, 0), 1 << 24, sink)
    t0 = time.perf_counter()
    nbytes = emit.emit_words(make_generator("philox", 1, 0), 1 << 30, sink)
    res["emit_raw_GBps"] = round(nbytes / (time.perf_counter() - t0) / 1e9, 2)

# §8(f) rank 3: snapshot records / checksum of 10M particles (cfg3 state)
from paper_2310_19925_b200 import brownian  # noqa: E402

cfg = brownian.SimConfig(10_000_000, 1)
p = brownian.init_particles(cfg)
t = timed(lambda: brownian._packed_records(p), reps=3)
res["pack_records_10M_to_host_s"] = round(t, 4)
t0 = time.perf_counter()
brownian.checksum(p)
res["checksum_10M_s"] = round(time.perf_counter() - t0, 3)
print(json.dumps(res))
