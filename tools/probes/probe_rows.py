"""Multi-stream rows of 256 words (2^22 streams), u32 and f32, GB/s, for one generator.

    python tools/probes/probe_rows.py threefry [--tuning]   (--tuning: the CBRNG_* knobs' build)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2310_19925_b200 import _lib  # noqa: E402

if "--tuning" in sys.argv:
    _lib.use_tuning_build()
    sys.argv.remove("--tuning")
alg = ("philox", "threefry", "squares", "tyche").index(sys.argv[1] if len(sys.argv) > 1 else "threefry")
L = _lib.lib()
s = int(torch.cuda.current_stream().cuda_stream)
out = torch.empty(1 << 30, dtype=torch.float32, device="cuda")


def run(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return round(4 * (1 << 30) / (e0.elapsed_time(e1) / reps) / 1e6, 1)


print(sys.argv[1] if len(sys.argv) > 1 else "threefry", "rows256 u32",
      run(lambda: _lib.check(L.cbrng_prefix_words(alg, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s), "u32")),
      "f32", run(lambda: _lib.check(L.cbrng_prefix_uniform_f32(alg, None, 0, None, 0, 1 << 22, 256, out.data_ptr(), s),
                                    "f32")))
