"""Time the Philox Box-Muller fill (configs[3] kernel) under tuning-build env sets.

    TUNE_SETS="CBRNG_BM_LAYOUT=0;CBRNG_BM_LAYOUT=5" python tools/tune_bm.py

Each set runs in a fresh process bound to libcbrng_b200_tuning.so; 2^29 pairs
(2 x 4 GiB of f64) per launch, CUDA events over 10 launches after a warm-up.
"""
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
P = 1 << 29
z0 = torch.empty(P, dtype=torch.float64, device="cuda"); z1 = torch.empty_like(z0)
fn = lambda: _lib.check(L.cbrng_normal2_f64(0, 42, 0, 0, None, P, z0.data_ptr(), z1.data_ptr(), None, s))
fn(); fn(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): fn()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"ms": round(ms, 4), "gbs": round(P * 16 / ms / 1e6, 1), "gvalues_s": round(2 * P / ms / 1e6, 1)}))
'''


def main():
    sets = [s for s in os.environ.get("TUNE_SETS", "CBRNG_BM_LAYOUT=0;CBRNG_BM_LAYOUT=5").split(";") if s]
    out = []
    for rep in range(int(os.environ.get("TUNE_REPS", "2"))):
        for st in sets:
            env = dict(os.environ)
            for kv in st.split(","):
                k, v = kv.split("=")
                env[k] = v
            r = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True,
                               timeout=600)
            res = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-800:]}
            res["set"] = st
            res["rep"] = rep
            out.append(res)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
