"""Property tests of the host-side logic (no GPU): shard maps, the long-stream
segment map, and the engine's position bookkeeping against the reference
engine itself (generators.py:227-406) when the reference package is importable
in this container (it is test-time only; the GPU box never reads it)."""

from __future__ import annotations

import os
import sys

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2310_19925_b200 import generators as G
from paper_2310_19925_b200 import sharding

REF_SRC = "/root/reference/pkg/src"


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 2**40), st.integers(1, 64), st.sampled_from([1, 2, 4, 16]))
def test_shard_range_partitions(n, world, align):
    spans = [sharding.shard_range(n, r, world, align) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (lo, hi), (lo2, _) in zip(spans, spans[1:]):
        assert lo <= hi == lo2
    for lo, hi in spans:
        assert lo % align == 0 and (hi % align == 0 or hi == n)


@settings(max_examples=300, deadline=None)
@given(st.data())
def test_stream_segments_cover_range(data):
    per = data.draw(st.sampled_from([1 << 30, 1 << 32, 7]))
    lo = data.draw(st.integers(0, 2**36))
    length = data.draw(st.integers(0, 2**33 if per > 7 else 200))
    hi = lo + length
    segs = sharding.stream_segments(lo, hi, per)
    pos = lo
    for s, off, k in segs:
        assert k > 0 and 0 <= off and off + k <= per
        assert s * per + off == pos
        pos += k
    assert pos == hi


@settings(max_examples=300, deadline=None)
@given(st.sampled_from(["philox", "threefry", "squares"]), st.integers(0, 2**33), st.integers(0, 2**33))
def test_advance_composes(alg, a, b):
    g1 = G.make_generator(alg, 5, 6)
    g1._advance(a)
    g1._advance(b)
    g2 = G.make_generator(alg, 5, 6)
    g2._advance(a + b)
    assert g1.state_bytes() == g2.state_bytes()


def _reference():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from cbrng import generators as R

    return R


@settings(max_examples=60, deadline=None)
@given(st.sampled_from(["philox", "threefry", "squares", "tyche"]), st.lists(st.integers(0, 9), max_size=12),
       st.integers(0, 2**64 - 1), st.integers(0, 2**32 - 1))
def test_position_bookkeeping_matches_reference_engine(alg, draws, seed, ctr):
    """n scalar draws leave the reference engine and ours in the same 18-byte
    state (our _advance is pure bookkeeping: no word is generated here)."""
    R = _reference()
    ref = R.make_generator(alg, seed, ctr)
    ours = G.make_generator(alg, seed, ctr)
    for n in draws:
        for _ in range(n):
            ref.next_u32()
        if alg == "tyche":
            ours._block_ctr = (ours._block_ctr + n) & G.MASK32  # Tyche's serial state is GPU-side
        else:
            ours._advance(n)
        assert ours.state_bytes() == ref.state_bytes()
