"""ctypes front end of the CPU oracle (oracle/cbrng_oracle.c).

TEST INFRASTRUCTURE ONLY — the checker, never the product. Imported by
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference).
Parity of this oracle with the reference package is pinned by
tests/test_oracle.py against fixtures frozen from the reference itself
(tests/golden/make_golden.py).

Function names follow the reference (`/root/reference/pkg/src/cbrng`); each
docstring cites the reference line restated by the C function it wraps.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libcbrng_oracle.so"
ALG = {"philox": 0, "threefry": 1, "squares": 2, "tyche": 3}

_lib = None


def build() -> Path:
    """Compile the oracle (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        u32p, u64p, f32p, f64p, u8p = (C.POINTER(t) for t in (C.c_uint32, C.c_uint64, C.c_float, C.c_double, C.c_uint8))
        L.orc_philox_block.argtypes = [u32p, u32p, u32p]
        L.orc_threefry_block.argtypes = [u32p, u32p, C.c_int, u32p]
        L.orc_squares_key.argtypes = [C.c_uint64]
        L.orc_squares_key.restype = C.c_uint64
        L.orc_squares_round.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_squares_round.restype = C.c_uint32
        L.orc_tyche_mix.argtypes = [u32p]
        L.orc_tyche_init.argtypes = [C.c_uint64, C.c_uint32, u32p]
        L.orc_words.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p, u32p]
        L.orc_prefix_words.argtypes = [C.c_int, u64p, C.c_uint64, u32p, C.c_uint32, C.c_uint64, C.c_uint32, u32p]
        L.orc_words_to_f32.argtypes = [u32p, C.c_uint64, f32p]
        L.orc_words_to_f64.argtypes = [u32p, C.c_uint64, f64p]
        L.orc_words_to_normal2.argtypes = [u32p, C.c_uint64, f64p, f64p]
        L.orc_uniform_f32.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, f32p]
        L.orc_brownian_init.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint32, f64p, f64p, f64p, f64p]
        L.orc_brownian_steps.argtypes = [C.c_int, C.c_uint64, u64p, f64p, f64p, f64p, f64p, C.c_uint32,
                                         C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double]
        L.orc_fnv1a64.argtypes = [u8p, C.c_uint64]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_brownian_checksum.argtypes = [C.c_uint64, u64p, f64p, f64p, f64p, f64p]
        L.orc_brownian_checksum.restype = C.c_uint64
        L.orc_digest_stream.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.orc_digest_stream.restype = C.c_uint64
        L.orc_digest_prefix.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int]
        L.orc_digest_prefix.restype = C.c_uint64
        L.orc_normal2_error.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, f64p, f64p,
                                        C.c_double, f64p]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray | None, t):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(t))


def _alg(a) -> int:
    if isinstance(a, str):
        return ALG[a.lower()]
    return int(a)


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(n)


def philox_block(key, ctr) -> tuple:
    """generators.py:101-122"""
    k = np.array(key, np.uint32); c = np.array(ctr, np.uint32); o = np.zeros(4, np.uint32)
    lib().orc_philox_block(_p(k, C.c_uint32), _p(c, C.c_uint32), _p(o, C.c_uint32))
    return tuple(int(x) for x in o)


def threefry_block(key, ctr, rounds: int = 20) -> tuple:
    """generators.py:125-154"""
    k = np.array(key, np.uint32); c = np.array(ctr, np.uint32); o = np.zeros(4, np.uint32)
    lib().orc_threefry_block(_p(k, C.c_uint32), _p(c, C.c_uint32), rounds, _p(o, C.c_uint32))
    return tuple(int(x) for x in o)


def squares_key(seed: int) -> int:
    """generators.py:157-170"""
    return int(lib().orc_squares_key(seed & 0xFFFFFFFFFFFFFFFF))


def squares_round(key: int, ctr: int) -> int:
    """generators.py:173-187"""
    return int(lib().orc_squares_round(key, ctr))


def tyche_mix(state) -> tuple:
    """generators.py:190-201"""
    s = np.array(state, np.uint32)
    lib().orc_tyche_mix(_p(s, C.c_uint32))
    return tuple(int(x) for x in s)


def tyche_init(seed: int, sc: int) -> tuple:
    """generators.py:204-218"""
    s = np.zeros(4, np.uint32)
    lib().orc_tyche_init(seed & 0xFFFFFFFFFFFFFFFF, sc & 0xFFFFFFFF, _p(s, C.c_uint32))
    return tuple(int(x) for x in s)


def stream_words(alg, seed: int, sc: int, n: int, block_ctr: int = 0, lane: int = 0,
                 tyche_state=None):
    """n x Generator.next_u32 from (block_ctr, lane) — generators.py:295-312, bulk.py:223-281.

    Returns the words (and, for Tyche with an explicit state, the final state).
    """
    a = _alg(alg)
    if a == 2:
        seed &= 0xFFFFFFFF
    out = np.empty(n, np.uint32)
    st = None if tyche_state is None else np.array(tyche_state, np.uint32)
    rc = lib().orc_words(a, seed & 0xFFFFFFFFFFFFFFFF, sc & 0xFFFFFFFF, block_ctr & 0xFFFFFFFF, lane, n,
                         _p(out, C.c_uint32), _p(st, C.c_uint32))
    if rc:
        raise ValueError("bad oracle arguments")
    if st is not None:
        return out, tuple(int(x) for x in st)
    return out


def prefix_words(alg, seeds, ctrs, nwords: int) -> np.ndarray:
    """bulk.py:162-207 (seeds/ctrs broadcast)."""
    seeds = np.atleast_1d(np.asarray(seeds, np.uint64))
    ctrs = np.atleast_1d(np.asarray(ctrs, np.uint32))
    seeds, ctrs = (np.ascontiguousarray(x) for x in np.broadcast_arrays(seeds, ctrs))
    n = seeds.shape[0]
    out = np.empty((n, nwords), np.uint32)
    lib().orc_prefix_words(_alg(alg), _p(seeds, C.c_uint64), 0, _p(ctrs, C.c_uint32), 0, n, nwords,
                           _p(out, C.c_uint32))
    return out


def prefix_words_arange(alg, seed_base: int, n: int, ctr: int, nwords: int) -> np.ndarray:
    out = np.empty((n, nwords), np.uint32)
    lib().orc_prefix_words(_alg(alg), None, seed_base, None, ctr, n, nwords, _p(out, C.c_uint32))
    return out


def words_to_f32(w: np.ndarray) -> np.ndarray:
    """distributions.py:105-107"""
    w = np.ascontiguousarray(w, np.uint32); o = np.empty(w.size, np.float32)
    lib().orc_words_to_f32(_p(w, C.c_uint32), w.size, _p(o, C.c_float))
    return o


def words_to_f64(w: np.ndarray) -> np.ndarray:
    """distributions.py:99-102"""
    w = np.ascontiguousarray(w, np.uint32); o = np.empty(w.size // 2, np.float64)
    lib().orc_words_to_f64(_p(w, C.c_uint32), o.size, _p(o, C.c_double))
    return o


def words_to_normal2(w: np.ndarray):
    """distributions.py:110-120"""
    w = np.ascontiguousarray(w, np.uint32); n = w.size // 4
    z0 = np.empty(n, np.float64); z1 = np.empty(n, np.float64)
    lib().orc_words_to_normal2(_p(w, C.c_uint32), n, _p(z0, C.c_double), _p(z1, C.c_double))
    return z0, z1


def uniform_f32(alg, seed: int, sc: int, n: int, out: np.ndarray | None = None) -> np.ndarray:
    """Fused CPU uniform_f32_array(make_generator(alg, seed, sc), n)."""
    a = _alg(alg)
    if a == 2:
        seed &= 0xFFFFFFFF
    o = np.empty(n, np.float32) if out is None else out
    lib().orc_uniform_f32(a, seed, sc, n, _p(o, C.c_float))
    return o


def uniform_f64(alg, seed: int, sc: int, n: int) -> np.ndarray:
    return words_to_f64(stream_words(alg, seed, sc, 2 * n))


def normal2(alg, seed: int, sc: int, n_pairs: int):
    return words_to_normal2(stream_words(alg, seed, sc, 4 * n_pairs))


def brownian_init(alg, n: int, init_ctr: int = 0, pid: np.ndarray | None = None):
    """brownian.py:112-126 -> (x, y, vx, vy)"""
    x, y, vx, vy = (np.empty(n, np.float64) for _ in range(4))
    pp = None if pid is None else np.ascontiguousarray(pid, np.uint64)
    lib().orc_brownian_init(_alg(alg), n, _p(pp, C.c_uint64), init_ctr & 0xFFFFFFFF,
                            *(_p(a, C.c_double) for a in (x, y, vx, vy)))
    return x, y, vx, vy


def brownian_steps(alg, state, first_it: int, nsteps: int, dt=0.01, gamma=0.1, mass=1.0,
                   init_ctr: int = 0, pid: np.ndarray | None = None):
    """brownian.py:129-142 iterated (in place on the four float64 arrays)."""
    x, y, vx, vy = state
    pp = None if pid is None else np.ascontiguousarray(pid, np.uint64)
    lib().orc_brownian_steps(_alg(alg), x.size, _p(pp, C.c_uint64), *(_p(a, C.c_double) for a in (x, y, vx, vy)),
                             init_ctr & 0xFFFFFFFF, first_it, nsteps, gamma, mass, dt)
    return state


def run_sim(alg, n: int, steps: int, dt=0.01, gamma=0.1, mass=1.0, init_ctr: int = 0):
    """brownian.py:164-195 (without timing) -> (x, y, vx, vy)"""
    st = brownian_init(alg, n, init_ctr)
    return brownian_steps(alg, st, 1, steps, dt, gamma, mass, init_ctr)


def fnv1a64(data) -> int:
    """_kernels.py:89-96"""
    b = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else np.ascontiguousarray(data).view(np.uint8).ravel()
    if b.size == 0:
        return 0xCBF29CE484222325
    b = np.ascontiguousarray(b)
    return int(lib().orc_fnv1a64(_p(b, C.c_uint8), b.size))


def brownian_checksum(x, y, vx, vy, pid: np.ndarray | None = None) -> int:
    """brownian.py:198-223"""
    arrs = [np.ascontiguousarray(a, np.float64) for a in (x, y, vx, vy)]
    pp = None if pid is None else np.ascontiguousarray(pid, np.uint64)
    return int(lib().orc_brownian_checksum(arrs[0].size, _p(pp, C.c_uint64), *(_p(a, C.c_double) for a in arrs)))


# ---------------------------------------------------------------------------
# Full-size checks (tests/test_gpu_fullsize.py): streamed digests and the
# Box-Muller error of a device array, never materialising the reference output.
# ---------------------------------------------------------------------------

def digest_stream(alg, seed: int, sc: int, word0: int, n: int, index0: int = 0, as_f32: bool = False) -> int:
    """sum_i mix64(mix64(index0 + i) ^ v_i) mod 2^64 over words (or their uniform f32 bit
    patterns) at positions [word0, word0 + n) of stream (seed, sc) (bulk.py:223-281)."""
    return int(lib().orc_digest_stream(_alg(alg), seed, sc, word0, n, index0, int(as_f32)))


def digest_prefix(alg, seed_base: int, n_streams: int, ctr: int, nwords: int, index0: int = 0,
                  as_f32: bool = False) -> int:
    """The same digest over prefix_words(alg, arange(seed_base, ...), ctr, nwords) (bulk.py:162-207)."""
    return int(lib().orc_digest_prefix(_alg(alg), seed_base, n_streams, ctr, nwords, index0, int(as_f32)))


def normal2_error(alg, seed: int, sc: int, bc0: int, z0: np.ndarray, z1: np.ndarray, tol: float = 4.0) -> dict:
    """Error of device Box-Muller pairs against the reference formula (distributions.py:72-81):
    max in ulp(max(|z|, 1)), max in ulps of z, and the count above `tol`."""
    z0 = np.ascontiguousarray(z0, np.float64)
    z1 = np.ascontiguousarray(z1, np.float64)
    out = np.zeros(3, np.float64)
    rc = lib().orc_normal2_error(_alg(alg), seed, sc, bc0, z0.size, _p(z0, C.c_double), _p(z1, C.c_double), tol,
                                 _p(out, C.c_double))
    if rc:
        raise ValueError("normal2_error: Philox/Threefry only")
    return {"max_units": float(out[0]), "max_rel_ulps": float(out[1]), "over_tol": int(out[2])}
