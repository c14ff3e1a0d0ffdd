"""A/B: the Philox, Threefry and Squares f32 fills of configs[1] back to back vs
one fused cbrng_uniform_f32_multi launch (and the Tyche rows after either).

    python tools/probes/probe_multi.py [reps]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2310_19925_b200 import _lib  # noqa: E402

N = 1 << 30
lib = _lib.lib()
outs = [torch.empty(N, dtype=torch.float32, device="cuda") for _ in range(4)]
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
algs = np.array([0, 1, 2], np.int32)
seeds = np.full(3, 42, np.uint64)
ctrs = np.zeros(3, np.uint32)
pos = np.zeros(3, np.uint64)
ns = np.full(3, N, np.uint64)
ptrs = np.array([o.data_ptr() for o in outs[:3]], np.uint64)


def seq():
    for i in range(3):
        _lib.check(lib.cbrng_uniform_f32(i, 42, 0, 0, None, N, outs[i].data_ptr(), None, sp), "f32")


def fused():
    _lib.check(lib.cbrng_uniform_f32_multi(3, algs.ctypes.data, seeds.ctypes.data, ctrs.ctypes.data,
                                           pos.ctypes.data, ns.ctypes.data, ptrs.ctypes.data, sp), "multi")


def tyche():
    _lib.check(lib.cbrng_prefix_uniform_f32(3, None, 0, None, 0, N // 256, 256, outs[3].data_ptr(), sp), "ty")


def t(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
res = {}
for k in range(2):
    res.setdefault("seq3_ms", []).append(round(t(seq, reps), 4))
    res.setdefault("fused3_ms", []).append(round(t(fused, reps), 4))
    res.setdefault("seq3+tyche_ms", []).append(round(t(lambda: (seq(), tyche()), reps), 4))
    res.setdefault("fused3+tyche_ms", []).append(round(t(lambda: (fused(), tyche()), reps), 4))
for k in list(res):
    res[k.replace("_ms", "_gsamples")] = round((4 if "tyche" in k else 3) * N / (min(res[k]) / 1e3) / 1e9, 1)
print(json.dumps(res))
