"""Time the configs[1] fills under code variants (env knobs read once per process).

Runs against the tuning build (`make -C paper_2310_19925_b200/csrc tuning`); the
product library has no knobs.

    python tools/tune_fills.py            # sweeps CBRNG_FILL_ILP x CBRNG_GRID_MULT x CBRNG_TF_VARIANT
    TUNE_SETS="CBRNG_CVT=1;CBRNG_CVT=3,CBRNG_CVT_MS=3" python tools/tune_fills.py   # explicit env sets
"""
import itertools
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_2310_19925_b200 import _lib
_lib.use_tuning_build()
L = _lib.lib(); s = int(torch.cuda.current_stream().cuda_stream)
N = 1 << 30
out = torch.empty(N, dtype=torch.float32, device="cuda")
res = {}
def run(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = {"ms": round(ms, 4), "gbs": round(N * 4 / ms / 1e6, 1)}
for a, nm in enumerate(["philox", "threefry", "squares"]):
    run(nm, lambda a=a: _lib.check(L.cbrng_uniform_f32(a, 42, 0, 0, None, N, out.data_ptr(), None, s)))
run("tyche_ms", lambda: _lib.check(L.cbrng_prefix_uniform_f32(3, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s)))
run("philox_ms_u32", lambda: _lib.check(L.cbrng_prefix_words(0, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s)))
run("memset", lambda: out.zero_())
z0 = torch.empty(1 << 27, dtype=torch.float64, device="cuda"); z1 = torch.empty_like(z0)
run("normal2_pairs", lambda: _lib.check(L.cbrng_normal2_f64(0, 42, 0, 0, None, 1 << 27, z0.data_ptr(), z1.data_ptr(), None, s)))
res["normal2_pairs"]["gbs"] = round(res["normal2_pairs"]["gbs"] / 2, 1)  # run() assumes 4 GiB; 2^27 pairs = 2 GiB
del z0, z1
import paper_2310_19925_b200 as cb
g = cb.make_generator("tyche", 42, 0)
g.words(1 << 16); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); w = g.words(1 << 22); e1.record(); e1.synchronize()
res["tyche_serial_mwords"] = {"gbs": round((1 << 22) / (e0.elapsed_time(e1) / 1e3) / 1e6, 1)}
del w
from paper_2310_19925_b200 import brownian
cfg = brownian.SimConfig(10_000_000, 200)
p = brownian.init_particles(cfg)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
brownian.run_steps(p, cfg); e0.record(); brownian.run_steps(p, cfg, start_iteration=201); e1.record(); e1.synchronize()
res["brownian_fused_psteps"] = {"gbs": round(10_000_000 * 200 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)}
cps = brownian.SimConfig(10_000_000, 100, mode="per_step")
brownian.run_steps(p, cps, start_iteration=401); e0.record(); brownian.run_steps(p, cps, start_iteration=501); e1.record(); e1.synchronize()
res["brownian_per_step_psteps"] = {"gbs": round(10_000_000 * 100 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)}
print(json.dumps(res))
'''

rows = []
if os.environ.get("TUNE_SETS"):
    # explicit env sets: "CBRNG_TF_VARIANT=4,CBRNG_CVT=3;CBRNG_CVT=1;..."
    sets = [dict(kv.split("=") for kv in grp.split(",") if kv) for grp in os.environ["TUNE_SETS"].split(";")]
else:
    GRID = [int(x) for x in os.environ.get("TUNE_GRID", "8").split(",")]
    ILPS = [int(x) for x in os.environ.get("TUNE_ILP", "16").split(",")]
    TFV = [int(x) for x in os.environ.get("TUNE_TF", "4").split(",")]
    sets = [{"CBRNG_FILL_ILP": str(i), "CBRNG_GRID_MULT": str(g), "CBRNG_TF_VARIANT": str(t)}
            for i, g, t in itertools.product(ILPS, GRID, TFV)]
for knobs in sets:
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-2000:])
        continue
    d = json.loads(r.stdout.strip().splitlines()[-1])
    rows.append((knobs, d))
    tag = " ".join(f"{k.replace('CBRNG_', '')}={v}" for k, v in knobs.items()) or "defaults"
    print(f"{tag}: " + " ".join(f"{k}={v['gbs']}" for k, v in d.items()), flush=True)
Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "tune_fills.json").write_text(json.dumps(rows, indent=1))
