"""D2H bandwidth into pinned host memory: one copy vs chunks spread over several streams."""
import json
import time

import torch

N = 1 << 30  # 4 GiB of f32
dev = torch.empty(N, dtype=torch.float32, device="cuda").fill_(1.0)
host = torch.empty(N, dtype=torch.float32, pin_memory=True)
res = {}
for nstreams in (1, 2, 4):
    for chunk_mb in (0, 64, 256):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        def run():
            if chunk_mb == 0 and nstreams == 1:
                host.copy_(dev, non_blocking=True)
                return
            c = (chunk_mb << 20) // 4 if chunk_mb else N // nstreams
            for i, o in enumerate(range(0, N, c)):
                with torch.cuda.stream(streams[i % nstreams]):
                    host[o:o + c].copy_(dev[o:o + c], non_blocking=True)
        run(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        res[f"streams={nstreams} chunk_mb={chunk_mb}"] = round(N * 4 / dt / 1e9, 1)
print(json.dumps(res, indent=1))
