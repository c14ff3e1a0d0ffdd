"""Raw stream emission at device rate: the B200 path
for `cbrng generate --format raw` (cli.py:84-100) and `fill_bytes`
(distributions.py:84-96), e.g. to feed PractRand / TestU01 through a pipe.

Chunks are generated into alternating device buffers and copied to pinned
host buffers asynchronously; while the GPU works on chunk k+1 the host writes
chunk k, so the sink (PCIe D2H, then the pipe/file) is the only bound.

    python -m paper_2310_19925_b200.emit --gen philox --seed 42 --counter 0 --n 1000000 > words.bin
"""

from __future__ import annotations

import argparse
import sys

import torch

from . import _dev
from .bulk import generator_fill
from .generators import Generator, make_generator

EMIT_CHUNK_WORDS = 1 << 24  # 64 MiB per chunk


def emit_words(g: Generator, n_words: int, sink, chunk_words: int = EMIT_CHUNK_WORDS) -> int:
    """Write the next n_words words of g (little-endian u32) to `sink` (a binary
    file-like object); advances g exactly like g.words(n_words). Returns bytes written."""
    if n_words < 0:
        raise ValueError("word count must be non-negative")
    if n_words == 0:
        return 0
    dev = _dev.cuda_device()
    k = min(chunk_words, n_words)
    dbuf = [torch.empty(k, dtype=torch.uint32, device=dev) for _ in range(2)]
    hbuf = [torch.empty(k, dtype=torch.uint32, pin_memory=True) for _ in range(2)]
    events = [torch.cuda.Event(), torch.cuda.Event()]
    pending = []  # (slot, count) in submission order
    written, done, slot = 0, 0, 0
    while done < n_words or pending:
        if done < n_words:
            m = min(k, n_words - done)
            generator_fill(g, m, "words", (dbuf[slot][:m],))
            hbuf[slot][:m].copy_(dbuf[slot][:m], non_blocking=True)
            events[slot].record()
            pending.append((slot, m))
            done += m
            slot ^= 1
        if len(pending) == 2 or done >= n_words:
            s, m = pending.pop(0)
            events[s].synchronize()
            sink.write(memoryview(hbuf[s].numpy()[:m].view("<u4")).cast("B"))
            written += 4 * m
    return written


def emit_bytes(g: Generator, n: int, sink) -> int:
    """fill_bytes(g, n) streamed to `sink`: ceil(n/4) words drawn, the last partial
    word truncated (distributions.py:84-96)."""
    if n < 0:
        raise ValueError("byte count must be non-negative")
    full, rem = divmod(n, 4)
    w = emit_words(g, full, sink)
    if rem:
        last = g.words(1, device="cpu").astype("<u4").tobytes()[:rem]
        sink.write(last)
        w += rem
    return w


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="raw little-endian u32 words of one stream to stdout")
    ap.add_argument("--gen", default="philox")
    ap.add_argument("--seed", type=lambda s: int(s, 0), default=0)
    ap.add_argument("--counter", type=lambda s: int(s, 0), default=0)
    ap.add_argument("--n", type=lambda s: int(s, 0), required=True, help="number of words")
    args = ap.parse_args(argv)
    try:
        g = make_generator(args.gen, args.seed, args.counter)
        emit_words(g, args.n, sys.stdout.buffer)
        sys.stdout.buffer.flush()
    except ValueError as exc:  # the reference CLI maps ValueError to exit 2 (cli.py:179-181)
        print(f"error: {exc}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
