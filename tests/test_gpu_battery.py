"""§8(f) rank 1: the statistical battery's data producers fused on the GPU
(cbrng_stream/prefix/buffer_byte_histogram, cbrng_avalanche,
cbrng_pearson_partials) against the reference's own reports
(tests/golden: run_battery, monobit/chi-square/KS on fixed blobs, avalanche,
interleave digests) and the CPU oracle."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import ALGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_19925_b200 import stats

    return stats


def test_histograms_exact(st, oracle):
    for alg in ALGS:
        for n in (1, 5, 4096, 100_003):
            c = st.histogram_stream(alg, 9, 2, n).cpu().numpy()
            ref = np.bincount(oracle.stream_words(alg, 9, 2, n).view(np.uint8), minlength=256)
            assert np.array_equal(c, ref), (alg, n)
    blob = np.random.default_rng(3).integers(0, 256, 100_007, dtype=np.uint8)
    assert np.array_equal(st.histogram_bytes(blob).cpu().numpy(), np.bincount(blob, minlength=256))


def test_interleave_histogram_matches_blob(st, oracle, golden):
    spec = st.InterleaveSpec(n_streams=1000, draws_per_stream=3, iterations=4)
    for alg in ALGS:
        blob = st.interleave_stream(spec, alg, 77)
        assert hashlib.sha256(blob).hexdigest() == golden["interleave_1000x3x4"][alg]
        c = st.interleave_histogram(spec, alg, 77).cpu().numpy()
        assert np.array_equal(c, np.bincount(np.frombuffer(blob, np.uint8), minlength=256))


def test_blob_reports(st, oracle, golden):
    blob = oracle.stream_words("squares", 3, 1, 100_003).astype("<u4").tobytes()[:400_010]
    assert st.report_to_dict(st.monobit(blob)) == golden["blob_tests"]["monobit"]
    assert st.report_to_dict(st.chi_square_bytes(blob)) == golden["blob_tests"]["chi_square_bytes"]
    u = oracle.uniform_f64("threefry", 5, 0, 10_000)
    assert st.report_to_dict(st.ks_uniform(u)) == golden["blob_tests"]["ks_uniform"]


@pytest.mark.parametrize("alg", ALGS)
def test_avalanche_exact(st, golden, alg):
    av = st.avalanche_stats(alg, 20_000)
    ref = golden["avalanche_20000"][alg]
    assert av.mean_hamming == ref["mean"] and av.z == ref["z"]
    assert av.bit_flip_rates.tolist() == ref["rates"]


@pytest.mark.parametrize("alg", ALGS)
def test_run_battery_matches_reference(st, golden, alg):
    """Every report of the reference's 16 MiB battery: integer-count statistics
    bit-identical; the correlation (sums vs numpy's two-pass corrcoef) to 1e-9."""
    got = [st.report_to_dict(r) for r in st.run_battery(alg, 16 * 2**20)]
    ref = golden["battery_16MiB"][alg]
    assert [g["test_name"] for g in got] == [r["test_name"] for r in ref]
    for g, r in zip(got, ref):
        assert g["verdict"] == r["verdict"] and g["n_samples"] == r["n_samples"]
        if g["test_name"] == "interstream_correlation":
            assert math.isclose(g["statistic"], r["statistic"], rel_tol=1e-9)
            assert math.isclose(g["p_value_or_z"], r["p_value_or_z"], rel_tol=1e-6)
        else:
            assert g == r, g["test_name"]
    assert st.battery_passes(st.run_battery(alg, 16 * 2**20))


@pytest.mark.parametrize("alg", ALGS)
def test_emit_words_and_bytes(st, oracle, alg):
    """§8(f) rank 2: raw emission == the stream's little-endian words; state advanced."""
    import io

    import paper_2310_19925_b200 as cb
    from paper_2310_19925_b200 import emit

    n = (1 << 16) + 5 if alg != "tyche" else 20_000
    g = cb.make_generator(alg, 5, 2)
    buf = io.BytesIO()
    assert emit.emit_words(g, n, buf, chunk_words=4099) == 4 * n
    ref = oracle.stream_words(alg, 5, 2, n + 3)
    assert buf.getvalue() == ref[:n].astype("<u4").tobytes()
    assert g.next_u32() == int(ref[n])
    g2 = cb.make_generator(alg, 5, 2)
    b2 = io.BytesIO()
    emit.emit_bytes(g2, 4 * n + 3, b2)
    assert b2.getvalue() == cb.fill_bytes(cb.make_generator(alg, 5, 2), 4 * n + 3)


def test_emit_cli_exit_codes(st):
    from paper_2310_19925_b200 import emit

    assert emit.main(["--gen", "nope", "--n", "4"]) == 2


# ---- foreign word sources: the reference's sabotage fixtures (fixtures.py:17-60),
# restated here as test infrastructure; the battery must take any word source
# (stats.py:289-318) and fail these exactly as the reference's battery does.
class _Constant:
    name, seed_bits = "constant", 64

    def stream_words(self, seed, stream_counter, n):
        return np.zeros(n, dtype=np.uint32)

    def prefix_words(self, seeds, stream_counters, nwords):
        n = np.broadcast_shapes(np.shape(np.atleast_1d(seeds)), np.shape(np.atleast_1d(stream_counters)))[0]
        return np.zeros((n, nwords), dtype=np.uint32)


class _CounterEcho:
    name, seed_bits = "counter-echo", 64

    def stream_words(self, seed, stream_counter, n):
        return (np.arange(n, dtype=np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)

    def prefix_words(self, seeds, stream_counters, nwords):
        n = np.broadcast_shapes(np.shape(np.atleast_1d(seeds)), np.shape(np.atleast_1d(stream_counters)))[0]
        return np.broadcast_to(np.arange(nwords, dtype=np.uint32), (n, nwords)).copy()


class _LowBitStuck:
    """A healthy Philox source (here: this package's own) with output bit 0 wedged at 1."""

    name, seed_bits = "low-bit-stuck", 64

    def __init__(self):
        from paper_2310_19925_b200.bulk import AlgorithmSource
        from paper_2310_19925_b200.generators import Algorithm

        self._inner = AlgorithmSource(Algorithm.PHILOX)

    def stream_words(self, seed, stream_counter, n):
        return np.asarray(self._inner.stream_words(seed, stream_counter, n, device="cpu")) | np.uint32(1)

    def prefix_words(self, seeds, stream_counters, nwords):
        return np.asarray(self._inner.prefix_words(seeds, stream_counters, nwords, device="cpu")) | np.uint32(1)


@pytest.mark.parametrize("name,cls", [("constant", _Constant), ("counter-echo", _CounterEcho),
                                      ("low-bit-stuck", _LowBitStuck)])
def test_run_battery_foreign_sources(st, name, cls):
    """Reports equal the reference battery's on its own sabotage fixtures
    (tests/golden/golden_r2.json, make_golden_r2.py)."""
    import json

    from conftest import GOLDEN_DIR

    ref = json.loads((GOLDEN_DIR / "golden_r2.json").read_text())["battery_sabotage_16MiB"][name]
    got = [st.report_to_dict(r) for r in st.run_battery(cls(), 16 * 2**20)]
    assert [g["test_name"] for g in got] == [r["test_name"] for r in ref]
    for g, r in zip(got, ref):
        assert g["verdict"] == r["verdict"] and g["n_samples"] == r["n_samples"], g["test_name"]
        for k in ("statistic", "p_value_or_z"):
            a, b = g[k], r[k]
            assert (math.isnan(a) and math.isnan(b)) or math.isclose(a, b, rel_tol=1e-9, abs_tol=1e-12), (g, r)
    assert not st.battery_passes(st.run_battery(cls(), 16 * 2**20))
