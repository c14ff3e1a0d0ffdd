#!/usr/bin/env python
"""Benchmark of the B200-native counter-based RNG hot path (BASELINE.json).

Headline (`value`, weak scaling): BASELINE configs[1] — uniform float32 fill of
2^30 values per GPU for each of the four generators (Philox/Threefry/Squares:
counter-parallel single streams; Tyche: 2^22 streams x 256, Tyche being serial
within a stream). One step = the four fills; value = samples/s over all ranks.
Rank r fills values [r 2^30, (r+1) 2^30) of the long-stream layout (value i is
word i mod P of stream (42, i div P), P = the stream's period: 2^34 words for
Philox/Threefry, 2^32 for Squares), so no rank repeats another's values.

Side rows (strong scaling: fixed totals split over the N ranks, each with an
order-free digest that must not depend on N):
  configs[2]  Brownian walk, 10M particles x 10k steps (pid-range shards),
              fused and per-step, against cuRAND Philox in the paper's shape;
  configs[3]  Box-Muller f64, 2^34 values (2^33 pairs, long-stream layout),
              against cuRAND's curandGenerateNormalDouble;
  configs[4]  10^8 Philox streams x 256 words (stream-range shards), against
              the cuRAND device API in the same shape;
each with its binding roofline (HBM and every compute pipe, the pipe work read
live from the loaded library's SASS, tools/sass_pipes.py) and, at N = 1, the
reference CPU path (C port, all host threads; and the reference package itself
from baseline/_ref when installed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--quick]
                    [--dist-backend nccl|gloo]

`--gpus N` without a launcher starts N ranks itself (torch.distributed.run,
127.0.0.1); under torchrun the launcher's RANK / WORLD_SIZE are used.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

METRIC = "Gsamples/s & HBM GB/s per generator; Brownian-walk particle-steps/s vs cuRAND"
ALGS = ["philox", "threefry", "squares", "tyche"]
N_PER_GPU = 1 << 30            # configs[1]: 2^30 f32 values per generator per GPU
TYCHE_STREAMS, TYCHE_WORDS = 1 << 22, 256
BR_PARTICLES, BR_STEPS = 10_000_000, 10_000          # configs[2] (total, split over ranks)
BM_PAIRS = 1 << 33                                   # configs[3]: 2^34 values = 2^33 pairs (total)
BM_CHUNK = 1 << 31                                   # pairs per launch group: 2 x 16 GiB buffers
MS_STREAMS, MS_WORDS = 100_000_000, 256              # configs[4] (total)
GOLDEN_R2 = ROOT / "tests" / "golden" / "golden_r2.json"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)", "sm_max_mhz": d.get("sm_max_mhz")}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


def golden() -> dict:
    return json.loads(GOLDEN_R2.read_text()) if GOLDEN_R2.exists() else {}


class ClockSampler:
    """SM clock + throttle reasons sampled every 5 ms by NVML during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, cuda_index: int):
        import threading

        self.cuda_index = cuda_index
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self.err = None

    def _handle(self, nv):
        import torch

        try:
            uuid = str(torch.cuda.get_device_properties(self.cuda_index).uuid)
            return nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def _run(self, nv, h):
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception as exc:  # keep timing even if NVML hiccups
                self.err = str(exc)
            self._stop.wait(0.005)

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._run, args=(nv, h), daemon=True)
            self._thread.start()
        except Exception as exc:
            self.err = str(exc)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        sm = [c for c, _ in self.samples]
        loaded = [c for c in sm if self.max_mhz and c > 0.5 * self.max_mhz] or sm
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "NVML, 5 ms"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run without a launcher: start N ranks under
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def host_threads() -> int:
    """Every host core this process may run on (torchrun sets OMP_NUM_THREADS=1 for
    its ranks; the CPU baselines run on rank 0 alone and take all the cores)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# Reference CPU path (test-infrastructure oracle: a C restatement of the
# reference algorithms, all host threads) — the `--impl reference` arm and the
# cpu_baseline legs. The reference package itself (numpy/numba) is timed too
# when baseline/_ref is installed (tools/ref_package_bench.py, a subprocess).
# ---------------------------------------------------------------------------

def cpu_reference(steps: int, warmup: int, quick: bool) -> dict:
    """configs[1] on the host: one step = the full per-GPU workload (4 x 2^30 f32 values;
    Tyche 2^22 streams x 256), about 2-3 s on 16 cores (--quick: 2^22 values)."""
    import numpy as np

    from oracle import oracle as orc

    orc.build()
    orc.set_num_threads(host_threads())
    threads = orc.num_threads()
    sample = N_PER_GPU if not quick else 1 << 22  # f32 values per generator per step
    ty_streams = sample // TYCHE_WORDS
    buf = np.empty(sample, np.float32)

    def one_step():
        for a in ALGS[:3]:
            orc.uniform_f32(a, 42, 0, sample, out=buf)
        w = orc.prefix_words_arange("tyche", 0, ty_streams, 0, TYCHE_WORDS)
        orc.words_to_f32(w.reshape(-1))

    for _ in range(max(warmup, 1)):
        one_step()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = time.perf_counter() - t0
    samples = steps * 4 * sample
    return {"value": samples / dt / 1e9, "unit": "Gsamples/s", "cores": threads, "kind": "port",
            "sample": f"{steps} step(s) x 4 generators x 2^{sample.bit_length() - 1} f32 values "
                      f"(Tyche: {ty_streams} streams x {TYCHE_WORDS}); oracle/cbrng_oracle.c, OpenMP {threads} threads",
            "seconds": dt}


def cpu_side_baselines(quick: bool) -> dict:
    """configs[2]/[3]/[4] on the host (C port, all threads), bounded samples."""
    from oracle import oracle as orc

    orc.set_num_threads(host_threads())
    threads = orc.num_threads()
    out = {}
    n, s = (200_000, 10) if quick else (2_000_000, 100)  # ~10 s on 16 cores
    t = time.perf_counter()
    st = orc.brownian_init("philox", n, 0)
    orc.brownian_steps("philox", st, 1, s)
    dt = time.perf_counter() - t
    out["configs[2]"] = {"value": n * s / dt, "unit": "particle-steps/s", "cores": threads, "kind": "port",
                         "sample": f"init + {s} steps of {n} particles (oracle brownian_init/steps, OpenMP)",
                         "seconds": round(dt, 3)}
    p = 1 << (20 if quick else 28)
    t = time.perf_counter()
    orc.normal2("philox", 42, 0, p)
    dt = time.perf_counter() - t
    out["configs[3]"] = {"value": 2 * p / dt / 1e9, "unit": "Gvalues/s", "cores": threads, "kind": "port",
                         "sample": f"2^{p.bit_length() - 1} Box-Muller pairs (oracle words + libm, OpenMP)",
                         "seconds": round(dt, 3)}
    r = 1 << (16 if quick else 22)
    t = time.perf_counter()
    orc.prefix_words_arange("philox", 0, r, 0, MS_WORDS)
    dt = time.perf_counter() - t
    out["configs[4]"] = {"value": r * MS_WORDS / dt / 1e9, "unit": "Gwords/s", "cores": threads, "kind": "port",
                         "sample": f"2^{r.bit_length() - 1} Philox streams x 256 (oracle prefix_words, OpenMP)",
                         "seconds": round(dt, 3)}
    return out


def reference_package(quick: bool) -> dict | None:
    """The reference package itself (baseline/_ref) on bounded samples, or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "cbrng").exists():
        return None
    env = dict(os.environ, PYTHONPATH=str(ref), NUMBA_CACHE_DIR="/tmp/numba_cache_ref")
    cmd = [sys.executable, str(ROOT / "tools" / "ref_package_bench.py")] + (["--quick"] if quick else [])
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as exc:  # reported, never the target
        return {"error": str(exc)[:300]}


def run_reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    m = cpu_reference(args.steps, args.warmup, args.quick)
    line = {"impl": "reference", "metric": METRIC, "value": m["value"], "unit": "Gsamples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["seconds"] / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "configs[1] uniform_f32 x4 generators (the full per-GPU workload per step; "
                                   "--quick: a 2^22-value sample)",
                       "sample": m["sample"]},
            "cpu_baseline": {"value": m["value"], "unit": "Gsamples/s", "cores": m["cores"], "kind": m["kind"],
                             "sample": m["sample"]},
            "e2e": {"value": m["value"], "unit": "Gsamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Rooflines
# ---------------------------------------------------------------------------

def roofline_of(work: dict | None, units_per_s: float, bytes_per_unit: float, pk: dict, sms: int, mhz: float) -> dict:
    """Fractions of HBM and of every compute pipe at this rate (per GPU); the
    binding roofline is the largest fraction."""
    import sass_pipes

    hbm = units_per_s * bytes_per_unit / 1e9
    fr = {"hbm": round(hbm / pk["hbm_gbs"], 3)}
    if work:
        fr.update(sass_pipes.fractions(work, units_per_s, sms, mhz))
    bound = max(fr, key=fr.get)
    out = {"bound": bound, "frac": fr[bound], "fractions": fr, "hbm_gbs": round(hbm, 1)}
    if work:
        out["per_unit"] = {k: work[k] for k in ("unit", "alu", "fma_heavy", "fp64", "xu", "issue") if k in work}
        out["kernel"] = work.get("kernel")
    return out


def headline_roofline(per_gen: dict, dom: str, pk: dict, sms: int, mhz: float, traffic) -> dict:
    """The contract's `roofline` for the dominant kernel, reported against its
    BINDING roofline (the largest of the HBM and pipe fractions)."""
    import sass_pipes

    r = per_gen[dom]["roofline"]
    b = r["bound"]
    if b == "hbm":
        achieved, peak, unit = r["hbm_gbs"], pk["hbm_gbs"], "GB/s"
        peak_src = pk["source"]
    else:
        ops = per_gen[dom]["roofline"]["per_unit"][b]
        achieved = round(ops * per_gen[dom]["gsamples_s"] * 1e9 / 1e12, 2)
        peak = round(sass_pipes.PIPE_RATE[b] * sms * mhz * 1e6 / 1e12, 2)
        unit = f"T thread-ops/s ({b} pipe)"
        peak_src = (f"{sass_pipes.PIPE_RATE[b]} thread-ops/clk/SM (profiles/r1s_probe_pipes.json) x {sms} SMs x "
                    f"{mhz:.0f} MHz (median SM clock in the timed region)")
    return {"bound": b, "achieved": achieved, "peak": peak, "unit": unit, "frac": r["frac"], "traffic": traffic,
            "kernel": r.get("kernel"), "fractions": r["fractions"],
            "hbm": {"achieved": r["hbm_gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": r["fractions"]["hbm"], "peak_source": pk["source"]},
            "per_unit": r.get("per_unit"), "peak_source": peak_src, "hbm_free": r.get("hbm_free"),
            "algorithmic_bytes_per_launch": N_PER_GPU * 4,
            "pipe_work_source": "tools/sass_pipes.py on the loaded libcbrng_b200.so (hot-loop SASS)"}


# ---------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the side rows (headline + e2e only)")
    ap.add_argument("--no-side", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines (tests)")
    ap.add_argument("--side-scale", type=int, default=1,
                    help="divide the side rows' totals by this (tests of the N-invariance logic; default 1 = BASELINE)")
    ap.add_argument("--dist-backend", default="nccl",
                    help="process-group backend (gloo lets the N>1 logic run several ranks on one GPU for testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2310_19925_b200 as cb
    import sass_pipes
    from paper_2310_19925_b200 import _lib, bulk, sharding

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    if world > ndev and args.dist_backend == "nccl":
        raise SystemExit(f"{world} ranks need {world} GPUs for NCCL ({ndev} visible); "
                         "use --dist-backend gloo to run the N>1 logic on fewer GPUs")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    lib = _lib.lib()
    so = str(_lib.LIB_PATH)
    stream = torch.cuda.current_stream(dev)
    sptr = int(stream.cuda_stream)
    pk = peaks()
    gold = golden()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, reps=1):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / 1e3 / reps)

    def all_ranks_true(ok: bool) -> bool:
        if world == 1:
            return ok
        t = torch.tensor([0 if ok else 1], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item()) == 0

    # ---------------- headline: configs[1] ----------------
    out = torch.empty(N_PER_GPU, dtype=torch.float32, device=dev)
    lo_val = rank * N_PER_GPU  # this rank's values of the long-stream layout
    ty_lo = rank * TYCHE_STREAMS

    def fill(alg: str):
        if alg == "tyche":
            _lib.check(lib.cbrng_prefix_uniform_f32(3, None, ty_lo, None, 0, TYCHE_STREAMS, TYCHE_WORDS,
                                                    out.data_ptr(), sptr), alg)
        else:
            sharding.uniform_f32_long(alg, 42, 0, lo_val, lo_val + N_PER_GPU, out)

    for _ in range(args.warmup):
        for a in ALGS:
            fill(a)
    ev = {a: [] for a in ALGS}
    barrier()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            for a in ALGS:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fill(a)
                e1.record(stream)
                ev[a].append((e0, e1))
        t1.record(stream)
        barrier()
    elapsed = max_over_ranks(t0.elapsed_time(t1) / 1e3)
    clocks = clk.summary()
    mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz") or 1965.0
    launches = 4 * args.steps
    value = 4 * N_PER_GPU * args.steps * world / elapsed / 1e9

    # full-array parity of this rank's range: the position-aware digest of every
    # value (untimed), against the digests the reference package itself produced
    # for configs[1] (tests/golden/make_golden_r2.py; rank 0's range = the N = 1 workload)
    ref_d = gold.get("cfg1_fullsize", {}).get("values", {})
    parity = {}
    for a in ALGS:
        fill(a)
        d = int(sharding.digest_words(out.view(torch.uint32), rank * N_PER_GPU if a != "tyche" else ty_lo * 256).item())
        parity[a] = f"{d & 0xFFFFFFFFFFFFFFFF:016x}"
    torch.cuda.synchronize(dev)

    work = {}
    for a in ALGS:
        try:
            work[a] = (sass_pipes.rows_work(so, 3, 1) if a == "tyche" else sass_pipes.fill_work(so, ALGS.index(a), 1))
        except Exception as exc:  # no cuobjdump on this host: HBM roofline only
            work[a] = None
            work_err = str(exc)
    per_gen = {}
    for a in ALGS:
        ms = max_over_ranks(statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev[a]))
        rate = N_PER_GPU / (ms / 1e3)
        per_gen[a] = {"ms": round(ms, 4), "gsamples_s": round(rate / 1e9, 2),
                      "roofline": roofline_of(work[a], rate, 4, pk, sms, mhz),
                      "digest": parity[a]}
        if rank == 0 and a in ref_d:
            per_gen[a]["matches_reference_fullsize"] = parity[a] == ref_d[a]
    # the Tyche layout (2^22 streams x 256, rows) reported for all four
    for a in ALGS[:3]:
        def rows(a=a):
            _lib.check(lib.cbrng_prefix_uniform_f32(ALGS.index(a), None, ty_lo, None, 0, TYCHE_STREAMS, TYCHE_WORDS,
                                                    out.data_ptr(), sptr), "rows")
        r_ms = timed(rows, reps=max(3, args.steps // 2)) * 1e3
        per_gen[a]["rows_layout"] = {"ms": round(r_ms, 4), "gsamples_s": round(N_PER_GPU / r_ms / 1e6, 2),
                                     "hbm_gbs": round(N_PER_GPU * 4 / r_ms / 1e6, 1),
                                     "what": "uniform f32, 2^22 streams (seeds r 2^22 + i, ctr 0) x 256 values, "
                                             "row-major: the Tyche layout of configs[1] (bulk.prefix_uniform_f32)"}
    per_gen["tyche"]["rows_layout"] = {"ms": per_gen["tyche"]["ms"], "gsamples_s": per_gen["tyche"]["gsamples_s"],
                                       "what": "the headline Tyche fill itself"}

    # HBM-free rate of the same kernels (libcbrng_ceiling.so: every store aimed at an
    # L2-resident ring): achieved / HBM-free near 1 means the fill runs at the rate
    # of its own instruction stream, whatever the HBM fraction says
    try:
        cl = _lib.ceiling_lib()
        for a in ALGS[:3]:
            def cfill(a=a):
                _lib.check(cl.cbrng_uniform_f32(ALGS.index(a), 42, 0, 0, None, N_PER_GPU, out.data_ptr(), None, sptr),
                           "ceiling fill")
            c_ms = timed(cfill, reps=max(3, args.steps // 2)) * 1e3
            per_gen[a]["roofline"]["hbm_free"] = {"ms": round(c_ms, 4),
                                                  "frac": round(c_ms / per_gen[a]["ms"], 3),
                                                  "what": "same kernel, stores into a 1 MB L2-resident ring "
                                                          "(libcbrng_ceiling.so); frac = HBM-free ms / ms"}
        def cty():
            _lib.check(cl.cbrng_prefix_uniform_f32(3, None, ty_lo, None, 0, TYCHE_STREAMS, TYCHE_WORDS, out.data_ptr(),
                                                   sptr), "ceiling rows")
        c_ms = timed(cty, reps=max(3, args.steps // 2)) * 1e3
        per_gen["tyche"]["roofline"]["hbm_free"] = {"ms": round(c_ms, 4), "frac": round(c_ms / per_gen["tyche"]["ms"], 3),
                                                    "what": "same kernel, rows of 2048-stream blocks into one 2 MB "
                                                            "L2-resident ring (libcbrng_ceiling.so); frac = HBM-free "
                                                            "ms / ms"}
    except (OSError, RuntimeError) as exc:  # ceiling build absent: the product numbers stand alone
        per_gen["philox"]["roofline"]["hbm_free_error"] = str(exc)[:200]
    dom = max(per_gen, key=lambda a: per_gen[a]["ms"])
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            summ = json.loads(prof.read_text())
            traffic = summ.get("traffic_bytes", {}).get(f"uniform_f32_{dom}")
        except (ValueError, AttributeError):
            traffic = None
    roofline = headline_roofline(per_gen, dom, pk, sms, mhz, traffic)

    line = {"metric": METRIC, "value": round(value, 3), "unit": "Gsamples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "configs[1]: uniform_f32 fill, 2^30 values x 4 generators per GPU "
                                   "(Philox/Threefry/Squares seed 42, long-stream layout; Tyche 2^22 streams x 256)",
                       "l2": "outputs 4 GiB per fill >> 126 MB L2 (no flush needed)",
                       "parallelism": f"value-range / stream-range shards x{world}, no collective",
                       "shards": "rank r: values [r 2^30, (r+1) 2^30) of stream counter r div 4 (Squares) "
                                 "or 0 (Philox/Threefry); Tyche streams [r 2^22, (r+1) 2^22)"},
            "roofline": roofline, "per_generator": per_gen, "gpu_launches": launches, "clocks": clocks}
    if ref_d and rank == 0:
        line["parity"] = {"fullsize_digests_match_reference": all(per_gen[a].get("matches_reference_fullsize")
                                                                  for a in ALGS),
                          "what": "rank 0's 4 x 2^30 outputs, position-aware digest vs the reference package's "
                                  "own outputs (tests/golden/golden_r2.json)"}
    if any(w is None for w in work.values()):
        line["roofline"]["pipe_work_error"] = work_err

    # write-only HBM ceiling for context (cudaMemsetAsync over the same 4 GiB)
    z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out.zero_()
    z0.record(stream)
    for _ in range(5):
        out.zero_()
    z1.record(stream)
    z1.synchronize()
    store_gbs = N_PER_GPU * 4 * 5 / (z0.elapsed_time(z1) / 1e3) / 1e9
    roofline["hbm"]["store_only_gbs"] = round(store_gbs, 1)

    # ---------------- e2e through the public API, host buffers ----------------
    del out
    torch.cuda.empty_cache()
    e2e_steps = 2
    host_out = torch.empty(N_PER_GPU, dtype=torch.float32, pin_memory=True)
    assert TYCHE_STREAMS * TYCHE_WORDS == N_PER_GPU

    def positioned(a: str):
        # the rank's range as the reference API expresses a position: an 18-byte
        # state (algorithm, seed, stream counter, block counter, cache position)
        per = sharding.words_per_stream(a)
        s, off = divmod(lo_val, per)
        g = cb.make_generator(a, 42, s)
        st = cb.Generator.from_state_bytes(g.state_bytes()[:13] + (off // g.words_per_block).to_bytes(4, "little")
                                           + b"\0")
        return st

    def e2e_step():
        for a in ALGS[:3]:
            cb.uniform_f32_array(positioned(a), N_PER_GPU, out=host_out)
        bulk.prefix_uniform_f32("tyche", range(ty_lo, ty_lo + TYCHE_STREAMS), 0, TYCHE_WORDS, out=host_out)

    e2e_step()
    barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    barrier()
    e2e_t = max_over_ranks(time.perf_counter() - t)
    line["e2e"] = {"value": round(4 * N_PER_GPU * e2e_steps * world / e2e_t / 1e9, 3), "unit": "Gsamples/s",
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * N_PER_GPU * 4,
                   "api": "uniform_f32_array(Generator.from_state_bytes(...), 2^30, out=pinned host) x3 + "
                          "bulk.prefix_uniform_f32(tyche, ..., out=pinned host)",
                   "note": "host-side wall clock, max over ranks; 64 MiB chunks with the D2H copy overlapped "
                           "(bulk.generator_fill -> _dev.pipelined_host_fill); bound by PCIe Gen5 x16 D2H "
                           "(56 GB/s measured, tools/probes/probe_d2h.py). The fills take scalar inputs only "
                           "(seed, counter), so there is nothing to copy host->device."}
    del host_out

    if not (args.quick or args.no_side):
        line["side"] = side_measurements(args, rank, world, dev, stream, lib, barrier, max_over_ranks, all_ranks_true,
                                         pk, gold, so, sms, mhz)

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference(1 if args.quick else 4, 1, args.quick)  # ~10 s of host work
            cpu.pop("seconds", None)
            line["cpu_baseline"] = cpu
            if not (args.quick or args.no_side):
                pkg = reference_package(args.quick)
                if pkg is not None:
                    line["cpu_baseline"]["reference_package"] = pkg.get("configs[1]", pkg)
                side_cpu = cpu_side_baselines(args.quick)
                for key, row in (("configs[2]", "brownian"), ("configs[3]", "box_muller_f64"),
                                 ("configs[4]", "multistream_words")):
                    cb_ = side_cpu[key]
                    if pkg is not None and key in pkg:
                        cb_["reference_package"] = {**pkg[key], "kind": "reference"}
                    line["side"][row]["cpu_baseline"] = cb_
        except Exception as exc:  # the baseline is reported, never the target
            line.setdefault("cpu_baseline", {"value": None, "error": str(exc)})
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def side_measurements(args, rank, world, dev, stream, lib, barrier, max_over_ranks, all_ranks_true, pk, gold, so,
                      sms, mhz) -> dict:
    import torch

    import sass_pipes
    from paper_2310_19925_b200 import _lib, brownian, sharding

    side = {}
    sptr = int(stream.cuda_stream)
    k = max(1, args.side_scale)
    BR_PARTICLES, BR_STEPS = globals()["BR_PARTICLES"] // k, max(globals()["BR_STEPS"] // k, 2)
    BM_PAIRS, MS_STREAMS = globals()["BM_PAIRS"] // k, globals()["MS_STREAMS"] // k
    n1_file = ROOT / "tests" / "golden" / "gpu_n1_digests.json"  # tools/record_n1_digests.py
    n1 = json.loads(n1_file.read_text()) if (k == 1 and n1_file.exists()) else {}

    def timed(fn, reps=1):
        fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / 1e3 / reps)

    def work_or_none(fn, *a):
        try:
            return fn(so, *a)
        except Exception:
            return None

    def invariant(key: str, digest: str) -> dict:
        ref = n1.get(key)
        return {"digest": digest, "n1_digest": ref, "gpu_count_invariant": (digest == ref) if ref else None}

    # ---- configs[2]: Brownian walk, 10M particles x 10k steps, pid-range shards (strong) ----
    lo, hi = sharding.shard_range(BR_PARTICLES, rank, world)
    n_loc = hi - lo
    cfg = brownian.SimConfig(BR_PARTICLES, BR_STEPS)
    p = brownian.init_particles(cfg, pid_base=lo, n=n_loc)
    x0 = [t.clone() for t in (p.x, p.y, p.vx, p.vy)]

    def reset():
        for t, s in zip((p.x, p.y, p.vx, p.vy), x0):
            t.copy_(s)

    res = {}
    digests = {}
    for mode in ("fused", "per_step"):
        reset()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        brownian.run_steps(p, brownian.SimConfig(BR_PARTICLES, BR_STEPS, mode=mode))
        e1.record(stream)
        barrier()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        res[mode] = {"seconds": round(t, 4), "psteps_per_s": BR_PARTICLES * BR_STEPS / t}
        acc = brownian.stats(p)
        sharding.allreduce_sum_(acc)
        digests[mode] = brownian.stats_summary(acc)
    stats = digests["fused"]
    del x0
    # cuRAND Philox, paper Fig. 2 shape (state in HBM), and a register-state variant
    cr = _lib.curand_lib()
    state = torch.empty(max(n_loc, 1) * cr.cbrng_curand_state_bytes(), dtype=torch.uint8, device=dev)
    for fused, name in ((0, "curand_per_step"), (1, "curand_fused")):
        cr.cbrng_curand_brownian_init(state.data_ptr(), n_loc, p.x.data_ptr(), p.y.data_ptr(), p.vx.data_ptr(),
                                      p.vy.data_ptr(), sptr)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cr.cbrng_curand_brownian_steps(state.data_ptr(), n_loc, p.x.data_ptr(), p.y.data_ptr(), p.vx.data_ptr(),
                                       p.vy.data_ptr(), BR_STEPS, 0.1, 1.0, 0.01, fused, sptr)
        e1.record(stream)
        barrier()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        res[name] = {"seconds": round(t, 4), "psteps_per_s": BR_PARTICLES * BR_STEPS / t}
    del state, p
    torch.cuda.empty_cache()
    fused_rate = res["fused"]["psteps_per_s"] / world
    side["brownian"] = {
        "config": f"configs[2]: {BR_PARTICLES} particles x {BR_STEPS} steps in total, pid-range shards over "
                  f"{world} GPU(s), Philox, pid = particle index, counter = step",
        "scaling": "strong",
        **{k: {"seconds": v["seconds"], "psteps_per_s": f"{v['psteps_per_s']:.4e}"} for k, v in res.items()},
        "speedup_fused_vs_curand_fused": round(res["fused"]["psteps_per_s"] / res["curand_fused"]["psteps_per_s"], 3),
        "speedup_vs_curand_per_step": round(res["per_step"]["psteps_per_s"] / res["curand_per_step"]["psteps_per_s"], 3),
        "speedup_fused_vs_curand_per_step": round(res["fused"]["psteps_per_s"] / res["curand_per_step"]["psteps_per_s"],
                                                  3),
        "roofline_fused": roofline_of(work_or_none(sass_pipes.brownian_fused_work), fused_rate, 0, pk, sms, mhz),
        "roofline_per_step": roofline_of(None, res["per_step"]["psteps_per_s"] / world, 64, pk, sms, mhz),
        "note_per_step": "64 B of HBM per particle-step (x, y, vx, vy read + written); at N >= 8 a shard's "
                         "state (<= 80 MB) fits in the 126 MB L2, so per-step strong scaling goes superlinear",
        "stats": stats,
        **invariant("cfg2_stats_digest", stats["digest"]),
        "modes_agree": digests["fused"]["digest"] == digests["per_step"]["digest"],
    }

    # ---- configs[3]: Box-Muller f64, 2^34 values = 2^33 pairs in total (strong) ----
    lo, hi = sharding.shard_range(BM_PAIRS, rank, world)
    chunk = min(BM_CHUNK, max(hi - lo, 1))
    z0 = torch.empty(chunk, dtype=torch.float64, device=dev)
    z1 = torch.empty(chunk, dtype=torch.float64, device=dev)
    pieces = [(c, min(c + chunk, hi)) for c in range(lo, hi, chunk)]

    def bm():
        for a, b in pieces:
            sharding.normal2_long("philox", 42, 0, a, b, z0[: b - a], z1[: b - a])

    t = timed(bm)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    for a, b in pieces:  # untimed verification pass: digest of every value
        sharding.normal2_long("philox", 42, 0, a, b, z0[: b - a], z1[: b - a])
        sharding.digest_words(z0[: b - a].view(torch.uint32), 2 * a, acc)
        sharding.digest_words(z1[: b - a].view(torch.uint32), 2 * BM_PAIRS + 2 * a, acc)
    sharding.allreduce_sum_(acc)
    bm_digest = f"{int(acc.item()) & 0xFFFFFFFFFFFFFFFF:016x}"
    # cuRAND Philox host API, the same 2^34 doubles (curandGenerateNormalDouble), this rank's share
    cr = _lib.curand_lib()
    g = cr.cbrng_curand_create(42, sptr)
    cr.cbrng_curand_set_offset(g, 4 * lo)

    def cu_bm():
        for a, b in pieces:
            _lib.check(0 if cr.cbrng_curand_normal_f64(g, z0.data_ptr(), b - a) == 0 else -3, "curand normal")
            _lib.check(0 if cr.cbrng_curand_normal_f64(g, z1.data_ptr(), b - a) == 0 else -3, "curand normal")

    t_cu = timed(cu_bm)
    cr.cbrng_curand_destroy(g)
    pairs_s = BM_PAIRS / t / world
    # HBM-free rate of the same Box-Muller kernel on one 2^29-pair launch (libcbrng_ceiling.so)
    bm_free = None
    try:
        cl = _lib.ceiling_lib()
        p29 = min(1 << 29, chunk)

        def one(L):
            _lib.check(L.cbrng_normal2_f64(0, 42, 0, 0, None, p29, z0.data_ptr(), z1.data_ptr(), None, sptr), "bm")

        t_p, t_c = timed(lambda: one(lib), reps=5), timed(lambda: one(cl), reps=5)
        bm_free = {"ms": round(t_c * 1e3, 4), "product_ms": round(t_p * 1e3, 4), "frac": round(t_c / t_p, 3),
                   "what": "one 2^29-pair launch, same kernel with stores into a 1 MB L2-resident ring "
                           "(libcbrng_ceiling.so); frac = HBM-free ms / product ms"}
    except (OSError, RuntimeError) as exc:
        bm_free = {"error": str(exc)[:200]}
    side["box_muller_f64"] = {
        "config": f"configs[3]: 2^34 normals (2^33 pairs) in total, long-stream layout, pair-range shards over "
                  f"{world} GPU(s)",
        "scaling": "strong",
        "seconds": round(t, 4), "gvalues_s": round(2 * BM_PAIRS / t / 1e9, 2),
        "roofline": {**roofline_of(work_or_none(sass_pipes.fill_work, 0, 3), pairs_s, 16, pk, sms, mhz),
                     "hbm_free": bm_free},
        "curand_normal_double": {"seconds": round(t_cu, 4), "gvalues_s": round(2 * BM_PAIRS / t_cu / 1e9, 2),
                                 "api": "curandGenerateNormalDouble, CURAND_RNG_PSEUDO_PHILOX4_32_10"},
        "speedup_vs_curand": round(t_cu / t, 3),
        **invariant("cfg3_digest", bm_digest),
    }
    del z0, z1
    torch.cuda.empty_cache()

    # ---- configs[4]: 1e8 streams x 256 words in total, stream-range shards (strong) ----
    lo, hi = sharding.shard_range(MS_STREAMS, rank, world)
    w = torch.empty(max(hi - lo, 1) * MS_WORDS, dtype=torch.uint32, device=dev)

    def ms():
        _lib.check(lib.cbrng_prefix_words(0, None, lo, None, 0, hi - lo, MS_WORDS, w.data_ptr(), sptr), "prefix")

    t = timed(ms, reps=3)
    d = sharding.digest_words(w[: (hi - lo) * MS_WORDS], lo * MS_WORDS)
    sharding.allreduce_sum_(d)
    ms_digest = f"{int(d.item()) & 0xFFFFFFFFFFFFFFFF:016x}"
    ref4 = gold.get("cfg4_fullsize", {}).get("philox") if k == 1 else None
    cr = _lib.curand_lib()
    t_cu = timed(lambda: _lib.check(0 if cr.cbrng_curand_rows(lo, hi - lo, MS_WORDS, w.data_ptr(), sptr) == 0 else -3,
                                    "curand rows"), reps=3)
    words_s = MS_STREAMS * MS_WORDS / t / world
    ms_free = None
    try:  # HBM-free rate of the same rows kernel (libcbrng_ceiling.so: rows into one L2-resident ring)
        cl = _lib.ceiling_lib()
        t_c = timed(lambda: _lib.check(cl.cbrng_prefix_words(0, None, lo, None, 0, hi - lo, MS_WORDS, w.data_ptr(),
                                                             sptr), "ceiling rows"), reps=3)
        ms_free = {"seconds": round(t_c, 4), "frac": round(t_c / t, 3),
                   "what": "same kernel, rows of 2048-stream blocks into one 2 MB L2-resident ring "
                           "(libcbrng_ceiling.so); frac = HBM-free time / time"}
    except (OSError, RuntimeError) as exc:
        ms_free = {"error": str(exc)[:200]}
    side["multistream_words"] = {
        "config": f"configs[4]: 1e8 Philox streams x 256 words in total, stream-range shards over {world} GPU(s)",
        "scaling": "strong",
        "seconds": round(t, 4), "gwords_s": round(MS_STREAMS * MS_WORDS / t / 1e9, 2),
        "roofline": {**roofline_of(work_or_none(sass_pipes.rows_work, 0, 0), words_s, 4, pk, sms, mhz),
                     "hbm_free": ms_free},
        "curand_rows": {"seconds": round(t_cu, 4), "gwords_s": round(MS_STREAMS * MS_WORDS / t_cu / 1e9, 2),
                        "api": "device API: curand_init(seed = stream, 0, 0) + curand4, one thread per stream"},
        "speedup_vs_curand": round(t_cu / t, 3),
        "digest": ms_digest, "reference_digest": ref4,
        "oracle_note": "reference_digest: the reference package's own prefix_words over all 1e8 x 256 words "
                       "(tests/golden/make_golden_r2.py)",
        "gpu_count_invariant": (ms_digest == ref4) if ref4 else None,
        "matches_reference_fullsize": (ms_digest == ref4) if ref4 else None,
    }
    del w
    torch.cuda.empty_cache()

    # ---- cuRAND host-API fill of the headline shape (same box) ----
    cr = _lib.curand_lib()
    out = torch.empty(N_PER_GPU, dtype=torch.float32, device=dev)
    g = cr.cbrng_curand_create(42, sptr)
    t = timed(lambda: cr.cbrng_curand_uniform_f32(g, out.data_ptr(), N_PER_GPU), reps=5)
    cr.cbrng_curand_destroy(g)
    side["curand_uniform_f32"] = {"gsamples_s": round(N_PER_GPU * world / t / 1e9, 2),
                                  "hbm_gbs": round(N_PER_GPU * 4 / t / 1e9, 1)}
    del out
    torch.cuda.empty_cache()
    return side


if __name__ == "__main__":
    main()
