"""Bulk engines on sm_100a: drop-in for `cbrng.bulk` (/root/reference/pkg/src/cbrng/bulk.py).

Every function here is a thin shim over one C-ABI entry point
(include/cbrng_b200.h); all generation happens in the CUDA kernels.
Device tensors in -> device tensors out; numpy/python inputs -> numpy out
(the reference's types), so vector helpers stay drop-in for host callers.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .generators import MASK32, Algorithm, Generator, as_algorithm

U32 = np.uint32
U64 = np.uint64


def _any_cuda(*xs) -> bool:
    return any(isinstance(x, torch.Tensor) and x.is_cuda for x in xs)


def _bcast(xs, dtypes):
    """Broadcast mixed inputs and move them to the device as contiguous arrays."""
    if _any_cuda(*xs):
        dev = next(x.device for x in xs if isinstance(x, torch.Tensor) and x.is_cuda)
        ts = [_dev.as_dev(x, dt, dev) for x, dt in zip(xs, dtypes)]
        ts = [t.reshape(-1) if t.dim() == 0 else t for t in ts]
        shape = torch.broadcast_shapes(*[t.shape for t in ts])
        return [t.expand(shape).contiguous() for t in ts], shape, True
    arrs = [np.asarray(x).astype(dt, copy=False) for x, dt in zip(xs, dtypes)]
    arrs = np.broadcast_arrays(*arrs)
    shape = arrs[0].shape
    return [_dev.as_dev(np.ascontiguousarray(a).reshape(-1), dt) for a, dt in zip(arrs, dtypes)], shape, False


def _ret(t: torch.Tensor, shape, on_device: bool):
    if on_device:
        return t.reshape(shape)
    return t.cpu().numpy().reshape(shape)


def philox4x32(c0, c1, c2, c3, k0, k1):
    """Vector Philox4x32-10 over broadcastable uint32 arrays (bulk.py:49-66)."""
    ts, shape, on_dev = _bcast((c0, c1, c2, c3, k0, k1), (U32,) * 6)
    n = int(np.prod(shape)) if len(shape) else 1
    ctr = torch.stack(ts[:4]).contiguous()
    key = torch.stack(ts[4:]).contiguous()
    out = torch.empty((4, n), dtype=torch.uint32, device=ctr.device)
    _lib.check(_lib.lib().cbrng_philox4x32(ctr.data_ptr(), key.data_ptr(), n, out.data_ptr(), _dev.sptr(out)),
               "philox4x32")
    return tuple(_ret(out[i], shape, on_dev) for i in range(4))


def threefry4x32(c0, c1, c2, c3, k0, k1, k2, k3, rounds: int = 20):
    """Vector Threefry4x32 over broadcastable uint32 arrays (bulk.py:69-92)."""
    ts, shape, on_dev = _bcast((c0, c1, c2, c3, k0, k1, k2, k3), (U32,) * 8)
    n = int(np.prod(shape)) if len(shape) else 1
    ctr = torch.stack(ts[:4]).contiguous()
    key = torch.stack(ts[4:]).contiguous()
    out = torch.empty((4, n), dtype=torch.uint32, device=ctr.device)
    _lib.check(_lib.lib().cbrng_threefry4x32(ctr.data_ptr(), key.data_ptr(), rounds, n, out.data_ptr(),
                                             _dev.sptr(out)), "threefry4x32")
    return tuple(_ret(out[i], shape, on_dev) for i in range(4))


def squares32(ctr, key):
    """Vector squares32 over broadcastable uint64 arrays (bulk.py:95-108)."""
    (c, k), shape, on_dev = _bcast((ctr, key), (U64, U64))
    n = int(np.prod(shape)) if len(shape) else 1
    out = torch.empty(n, dtype=torch.uint32, device=c.device)
    _lib.check(_lib.lib().cbrng_squares32(c.data_ptr(), k.data_ptr(), n, out.data_ptr(), _dev.sptr(out)), "squares32")
    return _ret(out, shape, on_dev)


def squares_keys(seeds):
    """Vectorised 32->64-bit odd key expansion (bulk.py:111-118)."""
    (s,), shape, on_dev = _bcast((seeds,), (U64,))
    n = int(np.prod(shape)) if len(shape) else 1
    out = torch.empty(n, dtype=torch.uint64, device=s.device)
    _lib.check(_lib.lib().cbrng_squares_keys(s.data_ptr(), n, out.data_ptr(), _dev.sptr(out)), "squares_keys")
    return _ret(out, shape, on_dev)


def tyche_mix(a, b, c, d, rounds: int = 1):
    """Vector quarter round(s) over broadcastable uint32 arrays (bulk.py:121-131)."""
    ts, shape, on_dev = _bcast((a, b, c, d), (U32,) * 4)
    n = int(np.prod(shape)) if len(shape) else 1
    st = torch.stack(ts).contiguous()
    _lib.check(_lib.lib().cbrng_tyche_mix(st.data_ptr(), n, rounds, _dev.sptr(st)), "tyche_mix")
    return tuple(_ret(st[i], shape, on_dev) for i in range(4))


def tyche_init(seeds, stream_counters):
    """Vectorised warm-up: one Tyche state per (seed, counter) lane (bulk.py:134-146)."""
    (s, c), shape, on_dev = _bcast((seeds, stream_counters), (U64, U32))
    n = int(np.prod(shape)) if len(shape) else 1
    st = torch.empty((4, n), dtype=torch.uint32, device=s.device)
    _lib.check(_lib.lib().cbrng_tyche_init(s.data_ptr(), 0, c.data_ptr(), 0, n, st.data_ptr(), _dev.sptr(st)),
               "tyche_init")
    return tuple(_ret(st[i], shape, on_dev) for i in range(4))


def tyche_advance_state(state, steps: int):
    """Apply `steps` quarter rounds to one state (bulk.py:149-159) on the device."""
    st = torch.tensor([[int(w) & MASK32] for w in state], dtype=torch.int64).to(torch.uint32)
    st = st.to(_dev.cuda_device()).contiguous()
    remaining = int(steps)
    while remaining > 0:
        chunk = min(remaining, MASK32)
        _lib.check(_lib.lib().cbrng_tyche_mix(st.data_ptr(), 1, chunk, _dev.sptr(st)), "tyche_mix")
        remaining -= chunk
    return tuple(int(v) for v in st.cpu().numpy().reshape(-1))


def tyche_words_from(state, n: int, device="cpu"):
    """n serial Tyche words continuing `state`; returns (words, final state)."""
    s_in = np.array([int(w) & MASK32 for w in state], np.uint32)  # read by the call (kernel parameter)
    out = _dev.empty(max(n, 1), torch.uint32)
    st_out = _dev.empty(4, torch.uint32)
    _lib.check(_lib.lib().cbrng_words(int(Algorithm.TYCHE), 0, 0, 0, s_in.ctypes.data, n, out.data_ptr(),
                                      st_out.data_ptr(), _dev.sptr(out)), "tyche words")
    final = tuple(int(v) for v in st_out.cpu().numpy())
    words = out[:n]
    return (words.cpu().numpy() if device == "cpu" else words), final


def stream_words(alg, seed: int, stream_ctr: int, word_pos: int, n: int, *, out=None, device=None):
    """n words of a counter-based stream starting at stream word `word_pos`."""
    alg = as_algorithm(alg)
    if alg is Algorithm.TYCHE:
        raise ValueError("Tyche is serial; use tyche_words_from")
    sink = _dev.Sink(n, torch.uint32, out, device)
    if n:
        _lib.check(_lib.lib().cbrng_words(int(alg), seed, stream_ctr & MASK32, word_pos, None, n,
                                          sink.dev.data_ptr(), None, _dev.sptr(sink.dev)), "words")
    return sink.finish()


def _prefix_args(seeds, stream_counters, device=None):
    """Returns (seed tensor | None, seed_base, ctr tensor | None, ctr_scalar, n)."""
    if isinstance(seeds, range) and seeds.step == 1:
        s_t, s_base, n_s = None, seeds.start, len(seeds)
    else:
        s_t = _dev.as_dev(np.atleast_1d(_dev.to_numpy(seeds)).astype(U64, copy=False).reshape(-1)
                          if not (isinstance(seeds, torch.Tensor) and seeds.is_cuda) else seeds.reshape(-1), U64, device)
        s_base, n_s = 0, s_t.numel()
    if np.ndim(stream_counters) == 0 and not isinstance(stream_counters, torch.Tensor):
        c_t, c_scalar, n_c = None, int(stream_counters) & MASK32, None
    else:
        c_t = _dev.as_dev(stream_counters, U32, device).reshape(-1)
        c_scalar, n_c = 0, c_t.numel()
        if c_t.numel() == 1 and n_s != 1:
            c_t, c_scalar, n_c = None, int(c_t.cpu().numpy()[0]), None
    n = n_s
    if n_c is not None and n_c != n_s:
        if n_s == 1:  # broadcast a single seed against many counters
            n = n_c
            if s_t is None:
                s_t = torch.full((n,), s_base, dtype=torch.int64).to(torch.uint64)
            s_t = s_t.expand(n).contiguous().to(c_t.device)
        else:
            raise ValueError(f"seeds ({n_s}) and stream_counters ({n_c}) do not broadcast")
    return s_t, s_base, c_t, c_scalar, n


def prefix_words(algorithm, seeds, stream_counters, nwords: int, *, out=None, device=None):
    """First `nwords` words of many streams (bulk.py:162-207) -> (n_streams, nwords) uint32.

    `seeds` may be a `range` (the np.arange pid layout) to avoid materialising it.
    """
    alg = as_algorithm(algorithm)
    if nwords < 0:
        raise ValueError("word count must be non-negative")
    s_t, s_base, c_t, c_scalar, n = _prefix_args(seeds, stream_counters, None if _dev.is_host(device) else device)
    sink = _dev.Sink(n * nwords, torch.uint32, None if out is None else out.reshape(-1) if isinstance(out, torch.Tensor) else out.reshape(-1), device)
    if n and nwords:
        _lib.check(_lib.lib().cbrng_prefix_words(int(alg), _dev.ptr(s_t), s_base, _dev.ptr(c_t), c_scalar, n, nwords,
                                                 sink.dev.data_ptr(), _dev.sptr(sink.dev)), "prefix_words")
    res = sink.finish()
    if out is not None:
        return out
    return res.reshape(n, nwords)


def prefix_uniform_f32(algorithm, seeds, stream_counters, nvalues: int, *, out=None, device=None):
    """uniform_f32 map of prefix_words, fused (one word per value)."""
    alg = as_algorithm(algorithm)
    s_t, s_base, c_t, c_scalar, n = _prefix_args(seeds, stream_counters, None if _dev.is_host(device) else device)
    host = _dev.pinned_host_target(None if out is None else out.reshape(-1) if isinstance(out, torch.Tensor) else out,
                                   n * nvalues, torch.float32, device) if nvalues else None
    if host is not None:
        # host destination, large fill: stream ranges generated in chunks, D2H overlapped
        fn = _lib.lib().cbrng_prefix_uniform_f32

        def launch(ptrs, first, count, st):
            sp = None if s_t is None else s_t.data_ptr() + 8 * first
            cp = None if c_t is None else c_t.data_ptr() + 4 * first
            _lib.check(fn(int(alg), sp, s_base + first, cp, c_scalar, count, nvalues, ptrs[0], st),
                       "prefix_uniform_f32")

        _dev.pipelined_host_fill(n, torch.float32, [host], launch, row=nvalues)
        return out if out is not None else host.numpy().reshape(n, nvalues)
    sink = _dev.Sink(n * nvalues, torch.float32, None if out is None else out.reshape(-1), device)
    if n and nvalues:
        _lib.check(_lib.lib().cbrng_prefix_uniform_f32(int(alg), _dev.ptr(s_t), s_base, _dev.ptr(c_t), c_scalar, n,
                                                       nvalues, sink.dev.data_ptr(), _dev.sptr(sink.dev)),
                   "prefix_uniform_f32")
    res = sink.finish()
    return out if out is not None else res.reshape(n, nvalues)


def first_words(algorithm, seeds, stream_counters, *, device=None):
    """First output word of each stream (bulk.py:210-212)."""
    return prefix_words(algorithm, seeds, stream_counters, 1, device=device)[:, 0]


def philox_block_lanes(seeds, stream_ctrs, block_ctr: int, *, device=None):
    """_kernels.philox_block_lanes (_kernels.py:54-86) -> (n, 4) uint32."""
    s = _dev.as_dev(seeds, U64)
    c = _dev.as_dev(stream_ctrs, U64)
    n = s.numel()
    sink = _dev.Sink(4 * n, torch.uint32, None, device)
    _lib.check(_lib.lib().cbrng_philox_block_lanes(s.data_ptr(), c.data_ptr(), block_ctr, n, sink.dev.data_ptr(),
                                                   _dev.sptr(sink.dev)), "philox_block_lanes")
    return sink.finish().reshape(n, 4)


# kind -> (C entry point, words per element, output dtype, number of outputs)
_FILL_FN = {
    "words": ("cbrng_words", 1, torch.uint32, 1),
    "f32": ("cbrng_uniform_f32", 1, torch.float32, 1),
    "f64": ("cbrng_uniform_f64", 2, torch.float64, 1),
    "normal2": ("cbrng_normal2_f64", 4, torch.float64, 2),
}


def generator_fill(g: Generator, n_elems: int, kind: str, outs=(None, None), device=None):
    """Shared engine of words / uniform_*_array / normal2_array: fill n elements
    (wpe words each) from g's current stream position with ONE kernel launch and
    advance g exactly as n*wpe next_u32 calls would (bulk.py:223-281).

    Returns one result (or two for normal2) as CUDA tensors, numpy arrays
    (device="cpu") or the caller's `outs`.
    """
    if n_elems < 0:
        raise ValueError("word count must be non-negative")
    fn_name, wpe, dtype, n_out = _FILL_FN[kind]
    if g.algorithm is not Algorithm.TYCHE:
        hosts = [_dev.pinned_host_target(outs[i] if i < len(outs) else None, n_elems, dtype, device)
                 for i in range(n_out)]
        if all(h is not None for h in hosts):
            # host destination, large fill: generate in chunks and overlap the D2H copies
            fn = getattr(_lib.lib(), fn_name)
            base = g._word_pos()

            def launch(ptrs, first, count, st):
                _lib.check(fn(int(g.algorithm), g.seed, g.stream_counter, base + first * wpe, None, count, *ptrs,
                              None, st), fn_name)

            _dev.pipelined_host_fill(n_elems, dtype, hosts, launch)
            g._advance(n_elems * wpe)
            res = [outs[i] if (i < len(outs) and outs[i] is not None) else hosts[i].numpy() for i in range(n_out)]
            return res[0] if n_out == 1 else tuple(res)
    sinks = [_dev.Sink(n_elems, dtype, outs[i] if i < len(outs) else None, device) for i in range(n_out)]
    if n_elems:
        fn = getattr(_lib.lib(), fn_name)
        st = _dev.sptr(sinks[0].dev)
        ptrs = [sk.dev.data_ptr() for sk in sinks]
        if g.algorithm is Algorithm.TYCHE:
            s_in = np.array(g._tyche_state, dtype=U32)  # logical state at the current position
            s_out = _dev.empty(4, torch.uint32, sinks[0].dev.device)
            _lib.check(fn(int(g.algorithm), 0, 0, 0, s_in.ctypes.data, n_elems, *ptrs, s_out.data_ptr(), st), fn_name)
            g._ty_state = tuple(int(v) for v in s_out.cpu().numpy())
            g._ty_base = g._ty_state
            g._ty_pending = np.empty(0, U32)
            g._ty_win = 0
            g._block_ctr = (g._block_ctr + n_elems * wpe) & MASK32
        else:
            _lib.check(fn(int(g.algorithm), g.seed, g.stream_counter, g._word_pos(), None, n_elems, *ptrs, None, st),
                       fn_name)
            g._advance(n_elems * wpe)
    res = [sk.finish() for sk in sinks]
    return res[0] if n_out == 1 else tuple(res)


_MULTI_FN = {"words": ("cbrng_words_multi", torch.uint32), "f32": ("cbrng_uniform_f32_multi", torch.float32)}


def fill_many(gens, n, kind: str = "f32", *, outs=None, device=None):
    """Batched Generator.words / uniform_f32_array: job i fills n[i] (or n) values
    from gens[i]'s current position and advances gens[i], in order, exactly as the
    per-generator calls would (bulk.py:223-281), through one C-ABI call
    (cbrng_uniform_f32_multi / cbrng_words_multi; CBRNG_MULTI=1 runs a Philox,
    a Threefry and a Squares job interleaved in one kernel). Tyche generators
    (serial streams) take the per-generator path. Returns a list of results
    like generator_fill's.
    """
    if kind not in _MULTI_FN:
        raise ValueError(f"kind must be one of {sorted(_MULTI_FN)}")
    gens = list(gens)
    ns = [int(n)] * len(gens) if np.isscalar(n) else [int(x) for x in n]
    if len(ns) != len(gens):
        raise ValueError("n must be a scalar or one count per generator")
    if any(x < 0 for x in ns):
        raise ValueError("word count must be non-negative")
    outs = [None] * len(gens) if outs is None else list(outs)
    if len(outs) != len(gens):
        raise ValueError("outs must have one entry per generator")
    fn_name, dtype = _MULTI_FN[kind]
    sinks = [None if g.algorithm is Algorithm.TYCHE else _dev.Sink(k, dtype, o, device)
             for g, k, o in zip(gens, ns, outs)]
    res: list = [None] * len(gens)
    jobs = []  # (index, alg, seed, ctr, word_pos, n, ptr)
    saved = {id(g): (g._cache_pos, g._block_ctr) for g in gens if g.algorithm is not Algorithm.TYCHE}
    for i, (g, k) in enumerate(zip(gens, ns)):
        if g.algorithm is Algorithm.TYCHE:
            continue
        jobs.append((i, int(g.algorithm), g.seed, g.stream_counter, g._word_pos(), k, sinks[i].dev.data_ptr()))
        g._advance(k)
    if jobs:
        m = len(jobs)
        a = np.array([j[1] for j in jobs], np.int32)
        sd = np.array([j[2] for j in jobs], U64)
        ct = np.array([j[3] for j in jobs], U32)
        wp = np.array([j[4] for j in jobs], U64)
        nn = np.array([j[5] for j in jobs], U64)
        pp = np.array([j[6] for j in jobs], U64)
        st = _dev.sptr(sinks[jobs[0][0]].dev)
        rc = getattr(_lib.lib(), fn_name)(m, a.ctypes.data, sd.ctypes.data, ct.ctypes.data, wp.ctypes.data,
                                          nn.ctypes.data, pp.ctypes.data, st)
        if rc != 0:
            for g in gens:
                if id(g) in saved:
                    g._cache_pos, g._block_ctr = saved[id(g)]
            _lib.check(rc, fn_name)
    for i, g in enumerate(gens):
        if g.algorithm is Algorithm.TYCHE:
            res[i] = generator_fill(g, ns[i], kind, (outs[i],), device)
        else:
            res[i] = sinks[i].finish()
    return res


def generator_words(g: Generator, n: int, *, out=None, device=None):
    """Implementation of Generator.words (bulk.py:223-281); advances g in place."""
    return generator_fill(g, n, "words", (out,), device)


class AlgorithmSource:
    """Adapter giving the statistical battery a uniform word-stream surface (bulk.py:284-296)."""

    def __init__(self, algorithm):
        self.algorithm = as_algorithm(algorithm)
        self.name = self.algorithm.name.lower()
        self.seed_bits = 32 if self.algorithm is Algorithm.SQUARES else 64

    def stream_words(self, seed: int, stream_counter: int, n: int, *, device=None):
        return Generator(self.algorithm, seed, stream_counter).words(n, device=device)

    def prefix_words(self, seeds, stream_counters, nwords: int, *, device=None):
        return prefix_words(self.algorithm, seeds, stream_counters, nwords, device=device)
