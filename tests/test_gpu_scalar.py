"""The scalar transport (cbrng_scalar, include/cbrng_b200.h): the reference's
scalar API (generators.py:101-224 block functions, 295-320 generator windows)
served by one-lane kernels through a mapped pinned buffer. Bit-exact against
the oracle, including the edge cases of each op."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M32, M64 = 0xFFFFFFFF, 0xFFFFFFFFFFFFFFFF


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_19925_b200 as cb

    return cb


KEYS = [(0, 0), (M32, M32), (0x12345678, 0x9ABCDEF0), (42, 0)]
CTRS = [(0, 0, 0, 0), (M32, M32, M32, M32), (1, 2, 3, 4), (0xDEADBEEF, 0, 7, M32)]


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("ctr", CTRS)
def test_philox_block(cb, oracle, key, ctr):
    assert tuple(cb.philox_block(key, ctr)) == tuple(oracle.philox_block(key, ctr))


@pytest.mark.parametrize("rounds", [0, 1, 13, 20, 32])
@pytest.mark.parametrize("ctr", CTRS)
def test_threefry_block(cb, oracle, ctr, rounds):
    key = (1, M32, 0x0BADF00D, 5)
    assert tuple(cb.threefry_block(key, ctr, rounds=rounds)) == tuple(oracle.threefry_block(key, ctr, rounds))


@pytest.mark.parametrize("seed", [0, 1, M32, 1 << 32, M64, 0x0123456789ABCDEF])
def test_squares_key_and_round(cb, oracle, seed):
    k = cb.squares_key(seed)
    assert k == oracle.squares_key(seed)
    for ctr in (0, 1, M32, 1 << 32, M64):
        assert cb.squares_round(k, ctr) == oracle.squares_round(k, ctr)


@pytest.mark.parametrize("seed,sc", [(0, 0), (M64, M32), (7, 3), (1 << 40, 12345)])
def test_tyche_init_and_mix(cb, oracle, seed, sc):
    s = cb.tyche_init(seed, sc)
    assert s == oracle.tyche_init(seed, sc)
    assert cb.tyche_mix(s) == oracle.tyche_mix(s)


@pytest.mark.parametrize("alg", ["philox", "threefry", "squares"])
@pytest.mark.parametrize("pos,n", [(0, 0), (0, 1), (1, 7), (3, 64), (2, 4099), ((1 << 34) - 5, 16), (17, 1 << 18)])
def test_stream_words(cb, oracle, alg, pos, n):
    from paper_2310_19925_b200 import _lib

    a = ["philox", "threefry", "squares"].index(alg)
    got = _lib.scalar(_lib.SCALAR_STREAM_WORDS, [a, 9, 4, pos], n)
    if alg == "squares":
        pos &= M32  # counter = word position mod 2^32 (bulk.py:268)
        ref = np.concatenate([oracle.stream_words(alg, 9, 4, n, block_ctr=pos)]) if n else np.empty(0, np.uint32)
    else:
        ref = oracle.stream_words(alg, 9, 4, n, block_ctr=(pos >> 2) & M32, lane=pos & 3) if n else \
            np.empty(0, np.uint32)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n", [0, 1, 3, 64, 1000])
def test_tyche_words(cb, oracle, n):
    from paper_2310_19925_b200 import _lib

    s = oracle.tyche_init(11, 2)
    r = _lib.scalar(_lib.SCALAR_TYCHE_WORDS, s, n + 4)
    ref, fin = oracle.stream_words("tyche", 0, 0, n, tyche_state=s) if n else (np.empty(0, np.uint32), s)
    assert np.array_equal(r[:n], ref) and tuple(int(v) for v in r[n:]) == tuple(fin)


@pytest.mark.parametrize("n", [0, 1, 63, 64, 1000])
def test_tyche_seed_words(cb, oracle, n):
    """A fresh Tyche stream's init state, first n words and final state in one call."""
    from paper_2310_19925_b200 import _lib

    r = _lib.scalar(_lib.SCALAR_TYCHE_SEED_WORDS, [0x0123456789ABCDEF, 77], n + 8)
    s = oracle.tyche_init(0x0123456789ABCDEF, 77)
    ref, fin = oracle.stream_words("tyche", 0, 0, n, tyche_state=s) if n else (np.empty(0, np.uint32), s)
    assert tuple(int(v) for v in r[:4]) == tuple(s)
    assert np.array_equal(r[4:4 + n], ref) and tuple(int(v) for v in r[4 + n:]) == tuple(fin)


def test_errors(cb):
    from paper_2310_19925_b200 import _lib

    with pytest.raises(ValueError):
        _lib.scalar(9, [], 1)  # unknown op
    with pytest.raises(ValueError):
        _lib.scalar(_lib.SCALAR_PHILOX_BLOCK, [1, 2, 3], 4)  # wrong arity
    with pytest.raises(ValueError):
        _lib.scalar(_lib.SCALAR_STREAM_WORDS, [0, 1, 2, 3], _lib.SCALAR_MAX_WORDS + 1)
    with pytest.raises(ValueError):
        _lib.scalar(_lib.SCALAR_STREAM_WORDS, [3, 1, 2, 3], 4)  # Tyche has no random access
    with pytest.raises(ValueError):
        cb.threefry_block((0, 0, 0, 0), (0, 0, 0, 0), rounds=-1)


def test_generator_windows_match_reference_order(cb, oracle):
    """next_u32 across several window refills (64, 128, ... words) and a mid-block
    resume equals the oracle's serial stream."""
    for alg in ("philox", "threefry", "squares", "tyche"):
        g = cb.make_generator(alg, 5, 6)
        got = [g.next_u32() for _ in range(64 + 128 + 256 + 3)]
        assert np.array_equal(np.array(got, np.uint32), oracle.stream_words(alg, 5, 6, len(got))), alg


def test_scalar_calls_from_threads(cb, oracle):
    """cbrng_scalar is reentrant: 8 host threads interleaving block functions and
    generator windows (the reference drives its nogil kernels from a thread pool,
    brownian.py:185-191) get the same results as serial calls."""
    from concurrent.futures import ThreadPoolExecutor

    def work(t):
        bad = 0
        for i in range(100):
            key, ctr = (t, i), (i, t, 7, 9)
            bad += tuple(cb.philox_block(key, ctr)) != tuple(oracle.philox_block(key, ctr))
            bad += cb.squares_round(cb.squares_key(t), i) != oracle.squares_round(oracle.squares_key(t), i)
        g = cb.make_generator(("philox", "threefry", "squares", "tyche")[t % 4], t, 3)
        got = np.array([g.next_u32() for _ in range(300)], np.uint32)
        bad += not np.array_equal(got, oracle.stream_words(g.algorithm.name.lower(), t, 3, 300))
        return bad

    with ThreadPoolExecutor(8) as ex:
        assert sum(ex.map(work, range(8))) == 0
