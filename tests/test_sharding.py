"""Host-side sharding logic and the N>1 path on CPU (gloo, world_size 2).

The data path has no collective: every element is a pure function of its
global index. These tests check that (a) the shard maps tile the index space
exactly, (b) per-shard work computed independently (here by the oracle, as a
stand-in for one GPU per rank) reduces through torch.distributed to the
single-process answer bit for bit — the GPU-count-invariance claim.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2310_19925_b200 import sharding


@pytest.mark.parametrize("n", [0, 1, 7, 1000, 2**30 + 3])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("align", [1, 4])
def test_shard_range_tiles_exactly(n, world, align):
    prev = 0
    for r in range(world):
        lo, hi = sharding.shard_range(n, r, world, align)
        assert lo == prev and lo <= hi
        if hi != n:
            assert lo % align == 0 and hi % align == 0
        prev = hi
    assert prev == n


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        sharding.shard_range(10, 2, 2)


def test_stream_segments_long_layout():
    per = sharding.PAIRS_PER_STREAM
    segs = sharding.stream_segments(per - 5, 2 * per + 7)
    assert segs == [(0, per - 5, 5), (1, 0, per), (2, 0, 7)]
    assert sum(k for _, _, k in segs) == per + 12
    assert sharding.pairs_per_stream("squares") == 1 << 30


def test_digest_is_order_free_and_position_aware():
    rng = np.random.default_rng(0)
    w = rng.integers(0, 2**32, 10_000, dtype=np.uint32)
    whole = sharding.digest_words_np(w, 0)
    parts = sum(sharding.digest_words_np(w[lo:hi], lo) for lo, hi in
                (sharding.shard_range(w.size, r, 3) for r in range(3))) % 2**64
    assert parts == whole
    swapped = w.copy()
    swapped[[10, 20]] = swapped[[20, 10]]
    assert sharding.digest_words_np(swapped, 0) != whole


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_2310_19925_b200 import sharding as sh

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # configs[4] layout, shortened: streams 0..4095 x 64 words, stream-range shards
        n, nw = 4096, 64
        lo, hi = sh.shard_range(n, rank, world)
        words = orc.prefix_words_arange("threefry", lo, hi - lo, 0, nw)
        u = sh.digest_words_np(words.reshape(-1), lo * nw)
        d = torch.tensor([u - (1 << 64) if u >= 1 << 63 else u], dtype=torch.int64)  # two's-complement view
        sh.allreduce_sum_(d)
        # configs[2] layout, shortened: pid-range shards of a Brownian run
        m = 1000
        plo, phi = sh.shard_range(m, rank, world)
        pid = np.arange(plo, phi, dtype=np.uint64)
        st = orc.brownian_init("squares", phi - plo, 0, pid=pid)
        orc.brownian_steps("squares", st, 1, 20, pid=pid)
        xs = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        xpad = torch.zeros(m, dtype=torch.float64)
        xpad[: phi - plo] = torch.from_numpy(st[0])
        dist.all_gather(xs, xpad)
        if rank == 0:
            xcat = np.concatenate([xs[r].numpy()[: sh.shard_range(m, r, world)[1] - sh.shard_range(m, r, world)[0]]
                                   for r in range(world)])
            q.put((int(d.item()) % 2**64, xcat))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world_matches_single_process(world):
    from oracle import oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    digest, xcat = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = orc.prefix_words_arange("threefry", 0, 4096, 0, 64)
    assert digest == sharding.digest_words_np(whole.reshape(-1), 0)
    ref = orc.run_sim("squares", 1000, 20)
    assert np.array_equal(xcat, ref[0])
