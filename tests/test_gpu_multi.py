"""Batched fills (bulk.fill_many / cbrng_uniform_f32_multi / cbrng_words_multi).

The fused multi-generator kernel must give exactly what the per-generator
calls give (bulk.py:223-281), which the oracle pins: every job is checked
bit-exact against the oracle's stream at the generator's position, over the
sizes and positions that exercise each path (tile remainders, trailing
partial units, mid-block starts that leave the fused kernel, Squares counter
wrap, duplicate generators, Tyche in the batch).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_19925_b200 as cb

    return cb


def host(t):
    return t.cpu().numpy()


def _expect(oracle, alg, seed, sc, pos, n, kind):
    """Oracle words for n values from absolute word position pos."""
    w = oracle.stream_words(alg, seed, sc, pos + n)[pos:]
    return w if kind == "words" else oracle.words_to_f32(w)


@pytest.mark.parametrize("kind", ["words", "f32"])
@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 383, 384, 512, 513, 12289, 98304 + 7, 1 << 20])
def test_three_generators_sizes(cb, oracle, kind, n):
    gens = [cb.make_generator("philox", 7, 1), cb.make_generator("threefry", 8, 2),
            cb.make_generator("squares", 9, 3)]
    got = cb.fill_many(gens, n, kind)
    for g0, out in zip(("philox", "threefry", "squares"), got):
        seed, sc = {"philox": (7, 1), "threefry": (8, 2), "squares": (9, 3)}[g0]
        assert np.array_equal(host(out), _expect(oracle, g0, seed, sc, 0, n, kind)), (g0, n)


@pytest.mark.parametrize("kind", ["words", "f32"])
def test_positions_duplicates_and_tyche(cb, oracle, kind):
    """Unequal sizes, generators resumed mid-block (off the fused path), the same
    generator twice (the second job continues where the first ended) and a Tyche
    generator in the batch."""
    ph = cb.make_generator("philox", 11, 0)
    tf = cb.make_generator("threefry", 12, 5)
    sq = cb.make_generator("squares", 13, 6)
    ty = cb.make_generator("tyche", 14, 7)
    [tf.next_u32() for _ in range(3)]  # mid-block: per-job launch
    [sq.next_u32() for _ in range(5)]
    sizes = [70001, 5003, 4096 * 9 + 2, 1000, 33333]
    got = cb.fill_many([ph, tf, sq, ty, ph], sizes, kind)
    assert np.array_equal(host(got[0]), _expect(oracle, "philox", 11, 0, 0, sizes[0], kind))
    assert np.array_equal(host(got[1]), _expect(oracle, "threefry", 12, 5, 3, sizes[1], kind))
    assert np.array_equal(host(got[2]), _expect(oracle, "squares", 13, 6, 5, sizes[2], kind))
    tw = oracle.stream_words("tyche", 14, 7, sizes[3])
    assert np.array_equal(host(got[3]), tw if kind == "words" else oracle.words_to_f32(tw))
    assert np.array_equal(host(got[4]), _expect(oracle, "philox", 11, 0, sizes[0], sizes[4], kind))
    # generators advanced exactly as the per-generator calls would
    assert ph.next_u32() == int(oracle.stream_words("philox", 11, 0, sizes[0] + sizes[4] + 1)[-1])
    assert sq.next_u32() == int(oracle.stream_words("squares", 13, 6, 5 + sizes[2] + 1)[-1])


def test_squares_counter_wrap_leaves_fused_path(cb, oracle):
    """A Squares job whose counters wrap mod 2^32 runs through the wrap-checking kernel."""
    import torch

    n = 40000
    start = (1 << 32) - 1000
    from paper_2310_19925_b200 import _lib

    lib = _lib.lib()
    outs = [torch.empty(n, dtype=torch.uint32, device="cuda") for _ in range(2)]
    algs = np.array([2, 0], np.int32)
    seeds = np.array([21, 22], np.uint64)
    ctrs = np.array([4, 4], np.uint32)
    pos = np.array([start, 16], np.uint64)
    ns = np.array([n, n], np.uint64)
    ptrs = np.array([o.data_ptr() for o in outs], np.uint64)
    rc = lib.cbrng_words_multi(2, algs.ctypes.data, seeds.ctypes.data, ctrs.ctypes.data, pos.ctypes.data,
                               ns.ctypes.data, ptrs.ctypes.data, None)
    assert rc == 0
    torch.cuda.synchronize()
    assert np.array_equal(outs[0].cpu().numpy(), oracle.stream_words("squares", 21, 4, n, block_ctr=start))
    assert np.array_equal(outs[1].cpu().numpy(), oracle.stream_words("philox", 22, 4, 16 + n)[16:])


def test_fused_kernel_matches(cb, oracle):
    """The default back-to-back launches (product library) and, when the tuning
    build exists, CBRNG_MULTI=1 (the fused multi-generator kernel, a tuning-only
    variant) give the oracle's words, over sizes that hit every remainder path."""
    import hashlib
    import json
    import os
    import subprocess
    import sys

    code = r"""
import sys, json, hashlib, numpy as np
sys.path.insert(0, %r)
if %r:
    from paper_2310_19925_b200 import _lib; _lib.use_tuning_build()
import paper_2310_19925_b200 as cb
res = []
for n in (1, 3, 5, 383, 513, 12289, 98311, 1 << 20):
    for kind in ("words", "f32"):
        gens = [cb.make_generator(a, 5, 5) for a in ("squares", "philox", "threefry")]
        got = cb.fill_many(gens, [n, n + 1, n + 2], kind)
        res.append([hashlib.sha256(g.cpu().numpy().tobytes()).hexdigest() for g in got])
print(json.dumps(res))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tuning = os.path.exists(os.path.join(root, "paper_2310_19925_b200", "_lib", "libcbrng_b200_tuning.so"))
    res = []
    for v in ("0", "1") if tuning else ("0",):
        r = subprocess.run([sys.executable, "-c", code % (root, v == "1")], env=dict(os.environ, CBRNG_MULTI=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    exp = []
    for n in (1, 3, 5, 383, 513, 12289, 98311, 1 << 20):
        for kind in ("words", "f32"):
            row = []
            for a, k in (("squares", n), ("philox", n + 1), ("threefry", n + 2)):
                w = oracle.stream_words(a, 5, 5, k)
                row.append(hashlib.sha256((w if kind == "words" else oracle.words_to_f32(w)).tobytes()).hexdigest())
            exp.append(row)
    for r in res:
        assert r == exp


def test_errors(cb):
    import torch

    from paper_2310_19925_b200 import _lib

    lib = _lib.lib()
    out = torch.empty(64, dtype=torch.float32, device="cuda")
    one = np.ones(1, np.uint64)
    for alg, code in ((3, -1), (7, -2)):
        a = np.array([alg], np.int32)
        p = np.array([out.data_ptr()], np.uint64)
        n = np.array([64], np.uint64)
        rc = lib.cbrng_uniform_f32_multi(1, a.ctypes.data, one.ctypes.data, None, one.ctypes.data, n.ctypes.data,
                                         p.ctypes.data, None)
        assert rc == code
    a = np.array([0], np.int32)
    p = np.array([out.data_ptr() + 4], np.uint64)
    n = np.array([16], np.uint64)
    assert lib.cbrng_uniform_f32_multi(1, a.ctypes.data, one.ctypes.data, None, one.ctypes.data, n.ctypes.data,
                                       p.ctypes.data, None) == -4
    assert lib.cbrng_uniform_f32_multi(0, None, None, None, None, None, None, None) == 0
    with pytest.raises(ValueError):
        cb.fill_many([cb.make_generator("philox", 1, 0)], [-1])
    with pytest.raises(ValueError):
        cb.fill_many([cb.make_generator("philox", 1, 0)], [1, 2])


def test_random_batches_match_oracle(cb, oracle):
    """Random batches (generators, positions, sizes, repeats) through fill_many equal
    the oracle's streams at each job's position; the same batches through the
    fused kernel are covered by test_fused_kernel_matches."""
    rng = np.random.default_rng(2310)
    algs = ("philox", "threefry", "squares", "tyche")
    for trial in range(12):
        gens, meta = [], []
        for _ in range(int(rng.integers(1, 6))):
            a = algs[int(rng.integers(0, 4))]
            seed, sc = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32))
            g = cb.make_generator(a, seed, sc)
            skip = int(rng.integers(0, 9))
            [g.next_u32() for _ in range(skip)]
            gens.append(g)
            meta.append((a, seed, sc, skip))
        # repeat one generator so a job continues its predecessor
        gens.append(gens[0])
        meta.append(meta[0])
        ns = [int(rng.integers(0, 20000)) for _ in gens]
        kind = "words" if trial % 2 else "f32"
        got = cb.fill_many(gens, ns, kind)
        consumed = {}
        for out, (a, seed, sc, skip), n, g in zip(got, meta, ns, gens):
            pos = consumed.get(id(g), skip)
            w = oracle.stream_words(a, seed, sc, pos + n)[pos:]
            consumed[id(g)] = pos + n
            assert np.array_equal(host(out), w if kind == "words" else oracle.words_to_f32(w)), (trial, a, pos, n)


@pytest.mark.parametrize("kind", ["words", "f32"])
def test_squares_fast_path_boundary(cb, oracle, kind):
    """The Squares fill takes the finite-difference kernel exactly when counters
    bc0 .. bc0 + 4 (n_units + 1) - 1 stay below 2^32 (cbrng_fill.cu launch_fill_k);
    fills that end exactly at, one unit past and well past that boundary all equal
    the oracle's wrapping stream (bulk.py:268)."""
    import torch

    from paper_2310_19925_b200 import _lib

    lib = _lib.lib()
    fn = lib.cbrng_words if kind == "words" else lib.cbrng_uniform_f32
    dt = torch.uint32 if kind == "words" else torch.float32
    n = 4 * 3000 + 3
    units = n // 4
    for start in ((1 << 32) - 4 * (units + 1), (1 << 32) - 4 * (units + 1) + 1, (1 << 32) - 4 * units,
                  (1 << 32) - 2 * n):
        out = torch.empty(n, dtype=dt, device="cuda")
        assert fn(2, 77, 9, start, None, n, out.data_ptr(), None, None) == 0
        torch.cuda.synchronize()
        w = oracle.stream_words("squares", 77, 9, n, block_ctr=start & 0xFFFFFFFF)
        ref = w if kind == "words" else oracle.words_to_f32(w)
        assert np.array_equal(out.cpu().numpy(), ref), start


def test_bench_gpu_count_invariance_gloo(tmp_path):
    """`python bench.py --gpus 2` with no launcher starts 2 ranks itself (gloo, both on
    this GPU); its line says n_gpus 2, and the strong-scaled side rows' digests
    (configs[2] stats, configs[3] normals, configs[4] words; totals / 64) equal the
    N = 1 run's — results do not depend on the GPU count."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lines = {}
    for n in (1, 2):
        cmd = [sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n), "--dist-backend", "gloo",
               "--steps", "1", "--warmup", "3", "--side-scale", "64", "--no-cpu"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=root)
        assert r.returncode == 0, r.stderr[-3000:]
        lines[n] = json.loads(r.stdout.strip().splitlines()[-1])
    assert lines[1]["n_gpus"] == 1 and lines[2]["n_gpus"] == 2
    for row in ("brownian", "box_muller_f64", "multistream_words"):
        assert lines[1]["side"][row]["digest"] == lines[2]["side"][row]["digest"], row
    assert lines[1]["side"]["brownian"]["modes_agree"] and lines[2]["side"]["brownian"]["modes_agree"]
    # rank 0's headline range is the N = 1 workload: same digests
    for a in ("philox", "threefry", "squares", "tyche"):
        assert lines[1]["per_generator"][a]["digest"] == lines[2]["per_generator"][a]["digest"], a
