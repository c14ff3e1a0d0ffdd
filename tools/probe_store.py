"""Write-only HBM ceiling on this B200: memset vs our store pattern, zero vs
incompressible data, resident grid vs oversubscribed grids."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19925_b200 import _lib  # noqa: E402

cr = _lib.curand_lib()
N = 1 << 32  # bytes
out = torch.empty(N // 4, dtype=torch.uint32, device="cuda")
s = int(torch.cuda.current_stream().cuda_stream)
sms = torch.cuda.get_device_properties(0).multi_processor_count


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); e1.synchronize()
    return round(N / (e0.elapsed_time(e1) / reps / 1e3) / 1e9, 1)


res = {"memset_zero": t(lambda: out.zero_()), "fill_0xA5": t(lambda: out.fill_(0xA5A5A5A5))}
for pat in (0, 1):
    for mult in (0, 2, 4, 16):
        blocks = 0 if mult == 0 else sms * 8 * mult
        res[f"probe_p{pat}_grid{'res' if mult == 0 else f'x{mult}'}"] = t(
            lambda b=blocks, p=pat: cr.cbrng_probe_store(out.data_ptr(), N, p, b, s))
print(json.dumps(res))
