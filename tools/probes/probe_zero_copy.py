"""Fill kernels writing straight into pinned host memory (zero-copy over PCIe) vs the
chunked device fill + D2H pipeline of bulk.generator_fill, for 2^30 f32 values.

    python tools/probes/probe_zero_copy.py
"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2310_19925_b200 as cb  # noqa: E402
from paper_2310_19925_b200 import _lib  # noqa: E402

N = 1 << 30
lib = _lib.lib()
host = torch.empty(N, dtype=torch.float32, pin_memory=True)
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
res = {}
for alg, name in enumerate(("philox", "threefry", "squares")):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.cbrng_uniform_f32(alg, 42, 0, 0, None, N, host.data_ptr(), None, sp), "zc")
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res.setdefault(f"{name}_zero_copy_gbs", []).append(round(N * 4 / (t1 - t0) / 1e9, 2))
    for rep in range(3):
        g = cb.make_generator(name, 42, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cb.uniform_f32_array(g, N, out=host)
        t1 = time.perf_counter()
        res.setdefault(f"{name}_pipelined_gbs", []).append(round(N * 4 / (t1 - t0) / 1e9, 2))
print(json.dumps(res))
