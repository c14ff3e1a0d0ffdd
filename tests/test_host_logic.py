"""Host-side engine bookkeeping (no GPU): stream position arithmetic, the
18-byte state format and argument validation mirror the reference engine
(generators.py:227-406, brownian.py:37-65) exactly."""

from __future__ import annotations

import struct

import pytest

from paper_2310_19925_b200 import generators as G
from paper_2310_19925_b200.brownian import SimConfig


def fresh(alg="philox", seed=1, ctr=2):
    return G.Generator(G.Algorithm.from_name(alg), seed, ctr)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 7, 8, 1001])
def test_advance_matches_reference_counters(n):
    # reference: after n next_u32 on a 4-word algorithm, block_ctr = ceil(n/4), cache_pos = n % 4
    g = fresh()
    g._advance(n)
    assert g._block_ctr == (n + 3) // 4 and g._cache_pos == n % 4
    assert g._word_pos() == n
    h = fresh("squares")
    h._advance(n)
    assert h._block_ctr == n and h._word_pos() == n


def test_advance_composes_and_wraps():
    g = fresh("threefry")
    g._advance(5)
    g._advance(6)
    assert (g._block_ctr, g._cache_pos) == (3, 3)
    g._block_ctr, g._cache_pos = 2**32 - 1, 0
    g._advance(9)  # crosses the 2^32 block wrap (generators.py:288)
    assert (g._block_ctr, g._cache_pos) == (2, 1)
    s = fresh("squares")
    s._block_ctr = 2**32 - 2
    s._advance(5)
    assert s._block_ctr == 3


def test_state_bytes_roundtrip_and_layout():
    g = fresh("threefry", 0x1122334455667788, 0x99AABBCC)
    g._advance(6)
    blob = g.state_bytes()
    assert len(blob) == 18
    assert struct.unpack("<BQIIB", blob) == (1, 0x1122334455667788, 0x99AABBCC, 2, 2)
    r = G.Generator.from_state_bytes(blob)
    assert (r._block_ctr, r._cache_pos, r._word_pos()) == (2, 2, 6)


def test_single_word_algorithms_reject_cache_pos():
    with pytest.raises(ValueError):
        G.Generator.from_state_bytes(struct.pack("<BQIIB", 2, 1, 2, 3, 1))


def test_squares_keeps_low_seed_bits_and_key_split():
    assert fresh("squares", 2**40 + 5).seed == 5
    g = fresh("philox", 0x0102030405060708, 9)
    assert g._key == (0x05060708, 0x01020304)
    t = fresh("threefry", 0x0102030405060708, 9)
    assert t._key == (0x05060708, 0x01020304, 9, 0)


def test_algorithm_names_and_errors():
    assert G.Algorithm.from_name(" Tyche ") is G.Algorithm.TYCHE
    with pytest.raises(ValueError):
        G.Algorithm.from_name("mt19937")
    with pytest.raises(ValueError):
        G.make_generator(7, 0, 0)
    assert G.Philox(3, 4).algorithm is G.Algorithm.PHILOX and G.Tyche(3).stream_counter == 0


def test_position_repr_matches_reference_formula():
    g = fresh()
    g._advance(7)
    assert g._position() == 7 and "position=7" in repr(g)


def test_simconfig_validation():
    for kw in (dict(n_particles=0), dict(steps=-1), dict(dt=-0.1), dict(gamma=-1.0), dict(mass=0.0),
               dict(threads=0), dict(mode="warp")):
        with pytest.raises(ValueError):
            SimConfig(**{**dict(n_particles=4, steps=1), **kw})
    assert SimConfig(4, 1, algorithm="tyche").algorithm is G.Algorithm.TYCHE


def test_micro_benchmark_validation():
    """bench.py:36-45 error behaviour (raised before any device work)."""
    from paper_2310_19925_b200 import micro_benchmark

    with pytest.raises(ValueError):
        micro_benchmark("philox", [0], repetitions=1)
    with pytest.raises(ValueError):
        micro_benchmark("philox", [1], repetitions=0)
    with pytest.raises(ValueError):
        micro_benchmark("nonsense", [1])


def test_bench_renderers():
    from paper_2310_19925_b200.microbench import BenchRow, bench_rows_csv, format_bench_table

    rows = [BenchRow("threefry", 1, 1500.0, 6.7e5), BenchRow("threefry", 10, 1600.0, 6.25e6)]
    table = format_bench_table(rows)
    assert "threefry" in table and "words/s" in table
    csv = bench_rows_csv(rows).splitlines()
    assert csv[0] == "algorithm,length,median_ns,words_per_second" and csv[1].startswith("threefry,1,1500,")


def test_rotl32():
    # generators.py:97-98
    assert G.rotl32(0x80000001, 1) == 0x00000003
    assert G.rotl32(0x12345678, 16) == 0x56781234
    assert G.rotl32(0xDEADBEEF, 31) == ((0xDEADBEEF >> 1) | (1 << 31)) & 0xFFFFFFFF
