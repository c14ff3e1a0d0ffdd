"""Fused Brownian kernel throughput (10M particles x 1000 steps) under the current env knobs
(tuning build: `make -C paper_2310_19925_b200/csrc tuning`)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19925_b200 import _lib, brownian  # noqa: E402

_lib.use_tuning_build()

res = {}
for alg in ("philox", "threefry", "squares", "tyche"):
    steps = 1000 if alg != "tyche" else 100
    cfg = brownian.SimConfig(10_000_000, steps, algorithm=alg)
    p = brownian.init_particles(cfg)
    brownian.run_steps(p, brownian.SimConfig(10_000_000, 10, algorithm=alg))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    brownian.run_steps(p, cfg, start_iteration=11)
    e1.record()
    e1.synchronize()
    res[alg] = f"{10_000_000 * steps / (e0.elapsed_time(e1) / 1e3):.3e}"
print(json.dumps(res))
