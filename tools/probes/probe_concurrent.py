"""A/B: the four configs[1] fills (Philox, Threefry, Squares f32 single stream;
Tyche f32 rows) back to back on one stream vs launched on separate streams so the
block scheduler mixes CTAs of different generators on each SM (pipe-bound
Threefry/Squares next to HBM-bound Philox/Tyche).

    python tools/probes/probe_concurrent.py [reps]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2310_19925_b200 import _lib  # noqa: E402

N = 1 << 30
lib = _lib.lib()
outs = [torch.empty(N, dtype=torch.float32, device="cuda") for _ in range(4)]
main = torch.cuda.current_stream()
side = [torch.cuda.Stream() for _ in range(4)]


def launch(i, s):
    p = int(s.cuda_stream)
    if i < 3:
        _lib.check(lib.cbrng_uniform_f32(i, 42, 0, 0, None, N, outs[i].data_ptr(), None, p), "f32")
    else:
        _lib.check(lib.cbrng_prefix_uniform_f32(3, None, 0, None, 0, N // 256, 256, outs[3].data_ptr(), p), "ty")


def seq(order=(0, 1, 2, 3)):
    for i in order:
        launch(i, main)


def conc(groups):
    """groups: tuple of tuples; each group runs back to back on its own stream."""
    ev = torch.cuda.Event()
    ev.record(main)
    for g, s in zip(groups, side):
        s.wait_event(ev)
        for i in g:
            launch(i, s)
    for s in side[: len(groups)]:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


def t(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    e1.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
res = {"seq": t(seq, reps)}
for name, g in {"4 streams": ((0,), (1,), (2,), (3,)), "ph+tf | sq+ty": ((0, 1), (2, 3)),
                "tf | ph+sq+ty": ((1,), (0, 2, 3)), "ph+ty | tf+sq": ((0, 3), (1, 2)),
                "tf+sq | ph+ty": ((1, 2), (0, 3))}.items():
    res[name] = t(lambda g=g: conc(g), reps)
for i, nm in enumerate(["philox", "threefry", "squares", "tyche"]):
    res["alone_" + nm] = t(lambda i=i: launch(i, main), reps)
res["seq"] = t(seq, reps)
print(json.dumps(res))
