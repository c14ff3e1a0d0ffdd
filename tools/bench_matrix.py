"""Every single-stream fill kind x generator, plus the multi-stream rows, on one GPU:
GB/s of output and Gvalues/s (CUDA events, 4 GiB outputs >> L2).

    python tools/bench_matrix.py > gpurun_out/bench_matrix.json
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19925_b200 import _lib  # noqa: E402

lib = _lib.lib()
s = int(torch.cuda.current_stream().cuda_stream)
BYTES = 1 << 32
buf = torch.empty(BYTES // 4, dtype=torch.float32, device="cuda")
buf2 = torch.empty(BYTES // 8, dtype=torch.float64, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {}
for a, name in enumerate(["philox", "threefry", "squares"]):
    n32 = BYTES // 4
    t = timed(lambda: _lib.check(lib.cbrng_words(a, 42, 0, 0, None, n32, buf.data_ptr(), None, s)))
    res[f"{name}_u32"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(n32 / t / 1e9, 1)}
    t = timed(lambda: _lib.check(lib.cbrng_uniform_f32(a, 42, 0, 0, None, n32, buf.data_ptr(), None, s)))
    res[f"{name}_f32"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(n32 / t / 1e9, 1)}
    n64 = BYTES // 8
    t = timed(lambda: _lib.check(lib.cbrng_uniform_f64(a, 42, 0, 0, None, n64, buf2.data_ptr(), None, s)))
    res[f"{name}_f64"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(n64 / t / 1e9, 1)}
    npairs = BYTES // 16
    z1 = buf.view(torch.float64)[:npairs]
    t = timed(lambda: _lib.check(lib.cbrng_normal2_f64(a, 42, 0, 0, None, npairs, buf2.data_ptr(), z1.data_ptr(), None, s)))
    res[f"{name}_normal2"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(2 * npairs / t / 1e9, 1)}
rows = BYTES // 4 // 256
for a, name in enumerate(["philox", "threefry", "squares", "tyche"]):
    t = timed(lambda: _lib.check(lib.cbrng_prefix_words(a, None, 0, None, 0, rows, 256, buf.data_ptr(), s)), reps=5)
    res[f"{name}_rows256_u32"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(BYTES / 4 / t / 1e9, 1)}
    t = timed(lambda: _lib.check(lib.cbrng_prefix_uniform_f32(a, None, 0, None, 0, rows, 256, buf.data_ptr(), s)), reps=5)
    res[f"{name}_rows256_f32"] = {"gbs": round(BYTES / t / 1e9, 1), "gvalues_s": round(BYTES / 4 / t / 1e9, 1)}
print(json.dumps(res, indent=1))
