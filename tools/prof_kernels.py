"""Launch each hot-path kernel once at benchmark size (for ncu captures).

    ncu --set full --clock-control none --import-source on -k regex:<kernel> -c <n> \
        -o gpurun_out/prof python tools/prof_kernels.py [which...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2310_19925_b200 import _lib, brownian  # noqa: E402

args = [x for x in sys.argv[1:] if not x.startswith("--")]
which = set(args) or {"fill", "tyche", "normal", "prefix", "brownian"}
if "--tuning" in sys.argv:  # the tuning build (CBRNG_* knobs)
    _lib.use_tuning_build()
lib = _lib.lib()
s = int(torch.cuda.current_stream().cuda_stream)
N = 1 << 30
out = torch.empty(N, dtype=torch.float32, device="cuda")
if "fill" in which:
    for alg in range(3):
        _lib.check(lib.cbrng_uniform_f32(alg, 42, 0, 0, None, N, out.data_ptr(), None, s))
if "squares" in which:
    _lib.check(lib.cbrng_uniform_f32(2, 42, 0, 0, None, N, out.data_ptr(), None, s))
if "threefry" in which:
    _lib.check(lib.cbrng_uniform_f32(1, 42, 0, 0, None, N, out.data_ptr(), None, s))
if "tyche" in which:
    _lib.check(lib.cbrng_prefix_uniform_f32(3, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s))
if "prefix" in which:
    _lib.check(lib.cbrng_prefix_words(0, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s))
del out
if "normal" in which:
    z0 = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    z1 = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    _lib.check(lib.cbrng_normal2_f64(0, 42, 0, 0, None, 1 << 28, z0.data_ptr(), z1.data_ptr(), None, s))
if "brownian" in which:
    cfg = brownian.SimConfig(10_000_000, 100)
    p = brownian.init_particles(cfg)
    brownian.run_steps(p, cfg)  # fused (brownian_fused_philox_kernel)
    brownian.run_steps(p, brownian.SimConfig(10_000_000, 2, mode="per_step"), start_iteration=101)
torch.cuda.synchronize()
print("done")
