"""Multi-GPU sharding of the hot path: one process per GPU, no data-path collective.

Every output element is a pure function of its global index (stream, word
position, pid), so work shards by contiguous ranges with zero communication:
  * single-stream fills  -> counter range (word positions), cut on 4-word unit
    boundaries so every shard starts block-aligned;
  * multi-stream fills   -> stream range (seed_base = first stream);
  * Brownian walk        -> pid range (brownian.py:158-161 `_slices` semantics).
The only collective is a small NCCL allreduce of int64 statistics / order-free
digests (integer sums mod 2^64: associative, so results are identical for any
GPU count — the paper's reproducibility claim, SPEC/brownian.py:1-13).

The long-stream layout (cfg4, 2^34 normals > one Philox stream's 2^32 blocks):
pair i comes from stream (seed, ctr0 + i // 2^32), block i mod 2^32
(README.md:23-24 "shard long workloads across stream counters").
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .generators import MASK32, Algorithm, as_algorithm

PAIRS_PER_STREAM = 1 << 32  # one Philox/Threefry block per Box-Muller pair


def pairs_per_stream(alg) -> int:
    """Box-Muller pairs one stream holds before its counter wraps: 2^32 blocks
    (Philox/Threefry) or 2^32 words = 2^30 pairs (Squares)."""
    return 1 << 30 if as_algorithm(alg) is Algorithm.SQUARES else PAIRS_PER_STREAM


def shard_range(n: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """Contiguous balanced [lo, hi) of n items for `rank`, boundaries multiples of `align`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = (n + align - 1) // align
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(lo_u * align, n), min(hi_u * align, n)


def words_per_stream(alg) -> int:
    """Words one stream holds before its counter wraps: 2^32 blocks x 4 words
    (Philox/Threefry) or 2^32 words (Squares)."""
    return 1 << 32 if as_algorithm(alg) is Algorithm.SQUARES else 1 << 34


def stream_segments(lo: int, hi: int, per_stream: int = PAIRS_PER_STREAM):
    """Split global element range [lo, hi) into (stream_offset, first_index_in_stream, count) pieces."""
    out = []
    i = lo
    while i < hi:
        s, off = divmod(i, per_stream)
        k = min(hi - i, per_stream - off)
        out.append((s, off, k))
        i += k
    return out


def normal2_long(alg, seed: int, ctr0: int, lo: int, hi: int, z0: torch.Tensor, z1: torch.Tensor) -> None:
    """Box-Muller pairs [lo, hi) of the long-stream layout into z0/z1 (device, len hi-lo)."""
    alg = as_algorithm(alg)
    if alg is Algorithm.TYCHE:
        raise ValueError("Tyche is serial; the long-stream layout needs a counter-based algorithm")
    lib = _lib.lib()
    st = _dev.sptr(z0)
    pos = 0
    per_stream = pairs_per_stream(alg)
    for s, off, k in stream_segments(lo, hi, per_stream):
        _lib.check(lib.cbrng_normal2_f64(int(alg), seed, (ctr0 + s) & MASK32, 4 * off, None, k,
                                         z0[pos:].data_ptr(), z1[pos:].data_ptr(), None, st), "normal2")
        pos += k


def uniform_f32_long(alg, seed: int, ctr0: int, lo: int, hi: int, out: torch.Tensor) -> None:
    """Values [lo, hi) of the long-stream uniform f32 layout into `out` (device, len hi-lo):
    value i is word i mod P of stream (seed, ctr0 + i // P), P = words_per_stream(alg),
    so a range past one stream's period continues on the next stream counter instead of
    wrapping onto values already produced (README.md:23-24)."""
    alg = as_algorithm(alg)
    if alg is Algorithm.TYCHE:
        raise ValueError("Tyche is serial; the long-stream layout needs a counter-based algorithm")
    lib = _lib.lib()
    st = _dev.sptr(out)
    pos = 0
    for s, off, k in stream_segments(lo, hi, words_per_stream(alg)):
        _lib.check(lib.cbrng_uniform_f32(int(alg), seed, (ctr0 + s) & MASK32, off, None, k, out[pos:].data_ptr(),
                                         None, st), "uniform_f32")
        pos += k


def digest_words(words: torch.Tensor, global_offset: int, acc: torch.Tensor | None = None) -> torch.Tensor:
    """acc (1 x int64, device) += order-free position-aware digest of `words` (uint32 view)."""
    w = words.reshape(-1)
    if w.dtype != torch.uint32:
        w = w.view(torch.uint32)
    if acc is None:
        acc = torch.zeros(1, dtype=torch.int64, device=w.device)
    _lib.check(_lib.lib().cbrng_digest_u32(w.data_ptr(), w.numel(), global_offset, acc.data_ptr(), _dev.sptr(w)),
               "digest")
    return acc


def allreduce_sum_(t: torch.Tensor) -> torch.Tensor:
    """In-place int64 SUM over ranks (NCCL on GPU tensors); identity without a process group."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def mix64_np(z: np.ndarray) -> np.ndarray:
    """Host restatement of the digest mixer (for tests / cross-checks)."""
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def digest_words_np(words: np.ndarray, global_offset: int) -> int:
    idx = np.arange(global_offset, global_offset + words.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum(mix64_np(mix64_np(idx) ^ words.astype(np.uint64)), dtype=np.uint64))


# ---------------------------------------------------------------------------
# Rank-local entry points (one process per GPU; `rank`/`world` from torchrun)
# ---------------------------------------------------------------------------

def uniform_f32_shard(alg, seed: int, stream_ctr: int, n_total: int, rank: int, world: int, out=None):
    """This rank's slice [lo, hi) of uniform_f32_array(make_generator(alg, seed, ctr), n_total):
    a contiguous counter range cut on 4-word boundaries, filled with no communication.
    Returns (lo, hi, tensor). Tyche is serial within a stream and cannot be cut."""
    alg = as_algorithm(alg)
    if alg is Algorithm.TYCHE:
        raise ValueError("Tyche is sequential within a stream; shard Tyche work across streams instead")
    lo, hi = shard_range(n_total, rank, world, align=4)
    t = out if out is not None else torch.empty(hi - lo, dtype=torch.float32, device=_dev.cuda_device())
    if hi > lo:
        _lib.check(_lib.lib().cbrng_uniform_f32(int(alg), seed, stream_ctr & MASK32, lo, None, hi - lo, t.data_ptr(),
                                                None, _dev.sptr(t)), "uniform_f32")
    return lo, hi, t


def prefix_words_shard(alg, n_streams: int, nwords: int, ctr: int, rank: int, world: int, seed_base: int = 0):
    """This rank's rows [lo, hi) of prefix_words(alg, arange(seed_base, seed_base + n_streams), ctr, nwords)."""
    from . import bulk

    lo, hi = shard_range(n_streams, rank, world)
    return lo, hi, bulk.prefix_words(alg, range(seed_base + lo, seed_base + hi), ctr, nwords)


def run_sim_shard(cfg, rank: int, world: int):
    """Brownian walk on this rank's pid range; returns (particles, stats) with the
    int64 statistics all-reduced over ranks (identical for any world size)."""
    from . import brownian

    lo, hi = shard_range(cfg.n_particles, rank, world)
    p = brownian.init_particles(cfg, pid_base=lo, n=hi - lo)
    if cfg.steps:
        brownian.run_steps(p, cfg)
    acc = brownian.stats(p) if hi > lo else torch.zeros(8, dtype=torch.int64, device=_dev.cuda_device())
    allreduce_sum_(acc)
    return p, acc
