#!/usr/bin/env python
"""Benchmark of the B200-native counter-based RNG hot path (BASELINE.json).

Headline (`value`): BASELINE configs[1] — uniform float32 fill of 2^30 values
for each of the four generators on one GPU (Philox/Threefry/Squares: one
stream, counter-parallel; Tyche: 2^22 streams x 256, Tyche being serial within
a stream). One step = the four fills; value = samples/s over all ranks.
Weak scaling: rank r fills counter range [r*2^30, (r+1)*2^30) of the same
streams (Tyche: stream range), so the global result is one long stream.

Side measurements on the same line: per-generator GB/s and roofline fraction,
the paper's Brownian walk (configs[2], 10M x 10k, fused and per-step, against
cuRAND Philox in the paper's Fig. 2 shape), Box-Muller f64 (configs[3]) and
multi-stream words (configs[4]), cuRAND host-API fills, the e2e number through
the public API with host buffers, and the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gsamples/s & HBM GB/s per generator; Brownian-walk particle-steps/s vs cuRAND"
ALGS = ["philox", "threefry", "squares", "tyche"]
N_PER_GPU = 1 << 30            # configs[1]: 2^30 f32 values per generator per GPU
TYCHE_STREAMS, TYCHE_WORDS = 1 << 22, 256
# INT-pipe work per output word of each headline fill, counted in the SASS main
# loop of the default kernel (tools/sass_pipes.py): ALU-pipe instructions
# (LOP3/SHF/IADD3/LEA/ISETP/...) or FMA-heavy slots (IMAD 1, IMAD.HI 2,
# IMAD.WIDE 2.5 — the measured rates, profiles/r1s_probe_pipes.json). The
# binding pipe is the one with more work per word.
INT_WORK_PER_WORD = {
    "philox": ("fma_heavy", 10.28, "16 IMAD.WIDE (x2.5) + 1 IMAD per 4-word block; ALU 5.6/word"),
    "threefry": ("alu", 20.10, "37 SHF.L.W + 39 LOP3 + 4 SHF.R per 4-word block; FMA-heavy 14.9 slots/word"),
    "squares": ("fma_heavy", 12.31, "2.3 IMAD.WIDE (x2.5) + IMAD.HI (x2) + 4.5 IMAD per word (round 1 by finite differences); ALU 8.3/word"),
    "tyche": ("alu", 9.76, "4 SHF.L.W + 4 LOP3 + 1 I2FP per word + staging, + the 20-mix warm-up per 256-word row"),
}
PIPE_LANES_PER_CLK_SM = {"alu": 63.3, "fma_heavy": 63.2}  # measured LOP3 / IMAD rates, profiles/r1s_probe_pipes.json


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)", "sm_max_mhz": d.get("sm_max_mhz")}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


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


def cpu_reference(steps: int, warmup: int, args) -> dict:
    """The reference's CPU path on the host cores: the C oracle (a restatement of
    the reference algorithms, oracle/cbrng_oracle.c) with all host threads, on a
    bounded sample of configs[1] per step. Returns a measurement dict."""
    import numpy as np

    from oracle import oracle as orc

    orc.build()
    threads = orc.num_threads()
    sample = 1 << 25 if not args.quick else 1 << 22  # f32 values per generator per step
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


def run_reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    m = cpu_reference(args.steps, args.warmup, args)
    line = {"impl": "reference", "metric": METRIC, "value": m["value"], "unit": "Gsamples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["seconds"] / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "configs[1] uniform_f32 x4 generators (bounded CPU sample)",
                       "sample": m["sample"]},
            "cpu_baseline": {"value": m["value"], "unit": "Gsamples/s", "cores": m["cores"], "kind": m["kind"],
                             "sample": m["sample"]},
            "e2e": {"value": m["value"], "unit": "Gsamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the side measurements")
    ap.add_argument("--no-side", action="store_true")
    ap.add_argument("--dist-backend", default="nccl",
                    help="process-group backend (gloo lets the N>1 logic run several ranks on one GPU for testing)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2310_19925_b200 as cb
    from paper_2310_19925_b200 import _lib, bulk, sharding

    rank, world, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = int(stream.cuda_stream)
    pk = peaks()

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

    # ---------------- headline: configs[1] ----------------
    out = torch.empty(N_PER_GPU, dtype=torch.float32, device=dev)
    word0 = rank * N_PER_GPU  # this rank's counter range of the shared stream
    ty_lo = rank * TYCHE_STREAMS

    def fill(alg: str):
        if alg == "tyche":
            rc = lib.cbrng_prefix_uniform_f32(3, None, ty_lo, None, 0, TYCHE_STREAMS, TYCHE_WORDS, out.data_ptr(), sptr)
        else:
            rc = lib.cbrng_uniform_f32(ALGS.index(alg), 42, 0, word0, None, N_PER_GPU, out.data_ptr(), None, sptr)
        _lib.check(rc, alg)

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
    launches = 4 * args.steps
    samples = 4 * N_PER_GPU * args.steps * world
    value = samples / elapsed / 1e9
    bytes_per_fill = N_PER_GPU * 4
    per_gen = {}
    for a in ALGS:
        ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev[a])
        gbs = bytes_per_fill / (ms / 1e3) / 1e9
        per_gen[a] = {"ms": round(ms, 4), "gsamples_s": round(N_PER_GPU / (ms / 1e3) / 1e9, 2),
                      "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / pk["hbm_gbs"], 3)}
    dom = max(per_gen, key=lambda a: per_gen[a]["ms"])
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            summ = json.loads(prof.read_text())
            traffic = summ.get("traffic_bytes", {}).get(f"uniform_f32_{dom}")
            # the INT-pipe side of the roofline, from the committed ncu capture:
            # the busiest of issue / ALU / FMA-heavy is the kernel's compute bound
            pats = {"philox": "fill_kernel<0, 1", "threefry": "fill_kernel<1, 1", "squares": "fill_kernel<2, 1",
                    "tyche": "staged_prefix_kernel<3, 1"}
            for a, pat in pats.items():
                k = next((k for k in summ.get("kernels", []) if pat in k["kernel"]), None)
                if k:
                    pipes = {"issue": k.get("issue_active_pct"), "alu": k.get("alu_pct"),
                             "fma_heavy": k.get("fmaheavy_pct")}
                    bind = max(pipes, key=lambda p_: pipes[p_] or 0)
                    per_gen[a]["ncu"] = {**{p_: round(v, 1) for p_, v in pipes.items() if v is not None},
                                         "binding_pipe": bind, "source": f"profiles/{summ.get('tag')}_ncu.md"}
        except (ValueError, AttributeError, KeyError):
            traffic = None
    roofline = {"bound": "hbm", "achieved": per_gen[dom]["hbm_gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": per_gen[dom]["hbm_frac"], "traffic": traffic, "kernel": f"fill_kernel<{dom}, f32>",
                "algorithmic_bytes_per_launch": bytes_per_fill, "peak_source": pk["source"]}
    if "ncu" in per_gen[dom]:
        # the slower of the two rooflines binds: for an INT-pipe-bound generator
        # (Threefry: ALU) report the pipe's utilisation from the committed ncu capture
        n = per_gen[dom]["ncu"]
        roofline["compute_roofline"] = {"pipe": n["binding_pipe"], "utilization_pct": n.get(n["binding_pipe"]),
                                        "source": n["source"]}
    # INT-pipe roofline per generator (live: words/s over the measured pipe rate
    # at the measured clock) and the fraction of the slower of the HBM-write and
    # INT-pipe rooflines (the larger of the two utilisations)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz") or 1965.0
    for a, (pipe, ops, how) in INT_WORK_PER_WORD.items():
        achieved = ops * N_PER_GPU / (per_gen[a]["ms"] / 1e3)
        peak = PIPE_LANES_PER_CLK_SM[pipe] * sms * mhz * 1e6
        per_gen[a]["int_roofline"] = {"pipe": pipe, "ops_per_word": ops, "frac": round(achieved / peak, 3)}
        per_gen[a]["binding_frac"] = round(max(per_gen[a]["hbm_frac"], achieved / peak), 3)
        if a == dom:
            roofline.setdefault("compute_roofline", {}).update({
                "pipe": pipe, "ops_per_word": ops, "ops_source": how,
                "achieved_gops": round(achieved / 1e9, 1), "peak_gops": round(peak / 1e9, 1),
                "frac": round(achieved / peak, 3),
                "peak_source": f"{PIPE_LANES_PER_CLK_SM[pipe]} thread-ops/clk/SM (profiles/r1s_probe_pipes.json) "
                               f"x {sms} SMs x {mhz:.0f} MHz (median SM clock in the timed region)"})

    line = {"metric": METRIC, "value": round(value, 3), "unit": "Gsamples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "configs[1]: uniform_f32 fill, 2^30 values x 4 generators per GPU "
                                   "(Philox/Threefry/Squares single stream seed 42 ctr 0; Tyche 2^22 streams x 256)",
                       "l2": "outputs 4 GiB per fill >> 126 MB L2 (no flush needed)",
                       "parallelism": f"counter/stream-range shards x{world}, no collective"},
            "roofline": roofline, "per_generator": per_gen, "gpu_launches": launches, "clocks": clocks}

    # write-only HBM ceiling for context (cudaMemsetAsync over the same 4 GiB)
    z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out.zero_()
    z0.record(stream)
    for _ in range(5):
        out.zero_()
    z1.record(stream)
    z1.synchronize()
    store_gbs = bytes_per_fill * 5 / (z0.elapsed_time(z1) / 1e3) / 1e9
    roofline["store_only_gbs"] = round(store_gbs, 1)
    roofline["frac_of_store_only"] = round(per_gen[dom]["hbm_gbs"] / store_gbs, 3)

    # ---------------- e2e through the public API, host buffers ----------------
    del out
    torch.cuda.empty_cache()
    e2e_steps = 2
    host_out = torch.empty(N_PER_GPU, dtype=torch.float32, pin_memory=True)
    assert TYCHE_STREAMS * TYCHE_WORDS == N_PER_GPU
    host_ty = host_out  # one 4 GiB pinned buffer per rank (8 ranks: 32 GiB of pinned host memory, not 64)

    def e2e_step():
        for a in ALGS[:3]:
            g = cb.make_generator(a, 42, 0)
            g._block_ctr = (word0 // 4) & 0xFFFFFFFF if a != "squares" else word0 & 0xFFFFFFFF
            cb.uniform_f32_array(g, N_PER_GPU, out=host_out)
        bulk.prefix_uniform_f32("tyche", range(ty_lo, ty_lo + TYCHE_STREAMS), 0, TYCHE_WORDS, out=host_ty)

    e2e_step()
    barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    barrier()
    e2e_t = max_over_ranks(time.perf_counter() - t)
    line["e2e"] = {"value": round(4 * N_PER_GPU * e2e_steps * world / e2e_t / 1e9, 3), "unit": "Gsamples/s",
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * N_PER_GPU * 4,
                   "api": "uniform_f32_array(make_generator(a, 42, 0), 2^30, out=pinned host) x3 + "
                          "bulk.prefix_uniform_f32(tyche, ..., out=pinned host)",
                   "note": "host-side wall clock; 64 MiB chunks with the D2H copy overlapped (bulk.generator_fill -> "
                           "_dev.pipelined_host_fill); bound by PCIe Gen5 x16 D2H (56 GB/s measured, tools/probes/probe_d2h.py)"}
    del host_out, host_ty

    if not (args.quick or args.no_side):
        line["side"] = side_measurements(args, rank, world, dev, stream, lib, barrier, max_over_ranks, pk)
        line["gpu_launches"] = launches

    if rank == 0 and world == 1:
        try:
            line["cpu_baseline"] = cpu_reference(1, 1, args)
            line["cpu_baseline"].pop("seconds", None)
        except Exception as exc:  # the baseline is reported, never the target
            line["cpu_baseline"] = {"value": None, "error": str(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def side_measurements(args, rank, world, dev, stream, lib, barrier, max_over_ranks, pk) -> dict:
    import torch

    from paper_2310_19925_b200 import _lib, brownian, sharding

    side = {}
    sptr = int(stream.cuda_stream)

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

    # ---- configs[2]: Brownian walk, 10M particles x 10k steps, pid-range shards ----
    n_part, n_steps = 10_000_000, 10_000
    lo, hi = rank * n_part, (rank + 1) * n_part  # weak scaling: each rank owns 10M pids
    cfg = brownian.SimConfig(n_part, n_steps)
    p = brownian.init_particles(cfg, pid_base=lo, n=hi - lo)
    x0 = [t.clone() for t in (p.x, p.y, p.vx, p.vy)]

    def reset():
        for t, s in zip((p.x, p.y, p.vx, p.vy), x0):
            t.copy_(s)

    res = {}
    for mode in ("fused", "per_step"):
        reset()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        brownian.run_steps(p, brownian.SimConfig(n_part, n_steps, mode=mode))
        e1.record(stream)
        barrier()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        res[mode] = {"seconds": round(t, 4), "psteps_per_s": n_part * n_steps * world / t}
    acc = brownian.stats(p)
    sharding.allreduce_sum_(acc)
    stats = brownian.stats_summary(acc)
    del x0
    # cuRAND Philox, paper Fig. 2 shape (state in HBM), and a register-state variant
    cr = _lib.curand_lib()
    state = torch.empty(n_part * cr.cbrng_curand_state_bytes(), dtype=torch.uint8, device=dev)
    for fused, name in ((0, "curand_per_step"), (1, "curand_fused")):
        cr.cbrng_curand_brownian_init(state.data_ptr(), n_part, p.x.data_ptr(), p.y.data_ptr(), p.vx.data_ptr(),
                                      p.vy.data_ptr(), sptr)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cr.cbrng_curand_brownian_steps(state.data_ptr(), n_part, p.x.data_ptr(), p.y.data_ptr(), p.vx.data_ptr(),
                                       p.vy.data_ptr(), n_steps, 0.1, 1.0, 0.01, fused, sptr)
        e1.record(stream)
        barrier()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        res[name] = {"seconds": round(t, 4), "psteps_per_s": n_part * n_steps * world / t}
    del state, p
    torch.cuda.empty_cache()
    per_step_bytes = 64  # x, y, vx, vy read + written per particle-step
    bw = res["per_step"]["psteps_per_s"] / world * per_step_bytes / 1e9
    side["brownian"] = {
        "config": "configs[2]: 10M particles x 10k steps per GPU, Philox, pid = particle index, counter = step",
        **{k: {"seconds": v["seconds"], "psteps_per_s": f"{v['psteps_per_s']:.4e}"} for k, v in res.items()},
        "speedup_vs_curand_per_step": round(res["per_step"]["psteps_per_s"] / res["curand_per_step"]["psteps_per_s"], 3),
        "speedup_fused_vs_curand_fused": round(res["fused"]["psteps_per_s"] / res["curand_fused"]["psteps_per_s"], 3),
        "speedup_fused_vs_curand_per_step": round(res["fused"]["psteps_per_s"] / res["curand_per_step"]["psteps_per_s"], 3),
        "per_step_hbm_gbs": round(bw, 1), "per_step_hbm_frac": round(bw / pk["hbm_gbs"], 3),
        "stats": stats,
    }

    # ---- configs[3]: Box-Muller f64, 2^34 values = 2^33 pairs per GPU ----
    pairs = (1 << 33)
    chunk = 1 << 31  # 16 GiB per output array per chunk keeps memory bounded
    z0 = torch.empty(chunk, dtype=torch.float64, device=dev)
    z1 = torch.empty(chunk, dtype=torch.float64, device=dev)
    base = rank * pairs

    def bm():
        for c in range(pairs // chunk):
            sharding.normal2_long("philox", 42, 0, base + c * chunk, base + (c + 1) * chunk, z0, z1)

    t = timed(bm)
    vals = 2 * pairs * world
    gbs = 2 * pairs * 8 / t / 1e9
    side["box_muller_f64"] = {"config": "configs[3]: 2^34 normals (2^33 pairs) per GPU, long-stream layout",
                              "seconds": round(t, 4), "gvalues_s": round(vals / t / 1e9, 2),
                              "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / pk["hbm_gbs"], 3)}
    acc = sharding.digest_words(z0[: 1 << 20].view(torch.uint32), 0)
    del z0, z1
    torch.cuda.empty_cache()

    # ---- configs[4]: 100M streams x 256 words per GPU (stream-range shards) ----
    n_str, nw = 100_000_000, 256
    w = torch.empty(n_str * nw, dtype=torch.uint32, device=dev)
    s_lo = rank * n_str

    def ms():
        _lib.check(lib.cbrng_prefix_words(0, None, s_lo, None, 0, n_str, nw, w.data_ptr(), sptr), "prefix")

    t = timed(ms)
    gbs = n_str * nw * 4 / t / 1e9
    d = sharding.digest_words(w, s_lo * nw)
    sharding.allreduce_sum_(d)
    side["multistream_words"] = {"config": "configs[4]: 1e8 Philox streams x 256 words per GPU",
                                 "seconds": round(t, 4), "gwords_s": round(n_str * nw * world / t / 1e9, 2),
                                 "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / pk["hbm_gbs"], 3),
                                 "digest": f"{int(d.item()) & 0xFFFFFFFFFFFFFFFF:016x}"}
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
