"""Single-stream fills of 2^30 values (u32 words and uniform f32), GB/s, for one generator.

    python tools/probes/probe_fill.py squares
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2310_19925_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "squares"
alg = ("philox", "threefry", "squares").index(name)
L = _lib.lib()
s = int(torch.cuda.current_stream().cuda_stream)
N = 1 << 30
out = torch.empty(N, dtype=torch.float32, device="cuda")


def run(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return round(4 * N / (e0.elapsed_time(e1) / reps) / 1e6, 1)


print(name, "u32", run(lambda: _lib.check(L.cbrng_words(alg, 42, 0, 0, None, N, out.data_ptr(), None, s), "w")),
      "f32", run(lambda: _lib.check(L.cbrng_uniform_f32(alg, 42, 0, 0, None, N, out.data_ptr(), None, s), "f")))
