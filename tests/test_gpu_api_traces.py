"""Replay of random API-call traces recorded from the reference package
(tests/golden/make_api_traces.py -> tests/golden/api_traces.json) through the
drop-in package on the GPU: every scalar and bulk result, and the 18-byte
generator state after every call, must equal the reference's — bit for bit for
integers, exact float maps and states; within 4 ulp(max(|z|,1)) for Box-Muller.
"""

from __future__ import annotations

import hashlib
import json
import struct
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TRACES = json.loads((Path(__file__).resolve().parent / "golden" / "api_traces.json").read_text())["traces"]
BM_ULP = 4


def h16(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def f64bits(x: float) -> str:
    return struct.pack("<d", float(x)).hex()


def close(got, ref) -> bool:
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return got.shape == ref.shape and bool(
        np.all(np.abs(got - ref) <= BM_ULP * np.spacing(np.maximum(np.abs(ref), 1.0))))


def run_op(cb, g, op, arg):
    if op == "next_u32":
        return g, g.next_u32()
    if op == "next_u64":
        return g, g.next_u64()
    if op == "words":
        w = np.asarray(g.words(arg, device="cpu"), np.uint32)
        return g, {"sha": h16(w.tobytes()), "head": [int(x) for x in w[:3]]}
    if op == "uniform_f32":
        return g, np.float32(cb.uniform_f32(g)).tobytes().hex()
    if op == "uniform_f64":
        return g, f64bits(cb.uniform_f64(g))
    if op == "uniform_f32_array":
        return g, h16(np.asarray(cb.uniform_f32_array(g, arg, device="cpu"), np.float32).tobytes())
    if op == "uniform_f64_array":
        return g, h16(np.asarray(cb.uniform_f64_array(g, arg, device="cpu"), np.float64).tobytes())
    if op == "normal2":
        return g, list(cb.normal2(g))
    if op == "normal2_array":
        z0, z1 = cb.normal2_array(g, arg, device="cpu")
        return g, [list(np.asarray(z0)), list(np.asarray(z1))]
    if op == "range_u32":
        return g, cb.range_u32(g, arg)
    if op == "fill_bytes":
        return g, cb.fill_bytes(g, arg).hex()
    if op == "draw_double2":
        d = cb.draw_double2(g)
        return g, [f64bits(d.x), f64bits(d.y)]
    if op == "copy":
        return g.copy(), None
    if op == "restore":
        return cb.Generator.from_state_bytes(g.state_bytes()), None
    raise ValueError(op)


@pytest.fixture(scope="module")
def cb():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2310_19925_b200 as cb

    return cb


@pytest.mark.parametrize("k", range(len(TRACES)))
def test_trace(cb, k):
    t = TRACES[k]
    g = cb.make_generator(t["alg"], t["seed"], t["ctr"])
    for i, s in enumerate(t["steps"]):
        g, res = run_op(cb, g, s["op"], s["arg"])
        where = f"{t['alg']} seed={t['seed']:#x} ctr={t['ctr']:#x} step {i} {s['op']}({s['arg']})"
        if s["op"] in ("normal2", "normal2_array"):
            assert close(res, s["res"]), where
        else:
            assert res == s["res"], where
        assert g.state_bytes().hex() == s["state"], where


BULK = json.loads((Path(__file__).resolve().parent / "golden" / "api_traces.json").read_text())["bulk"]


def _sha32(x) -> str:
    return h16(np.ascontiguousarray(np.asarray(x), np.uint32).tobytes())


@pytest.mark.parametrize("k", range(len(BULK)))
def test_bulk_call(cb, k):
    """Multi-stream and vector entry points (bulk.py:49-296) on recorded inputs."""
    from paper_2310_19925_b200 import bulk

    c = BULK[k]
    u64 = lambda xs: np.asarray(xs, dtype=np.uint64)  # noqa: E731
    u32 = lambda xs: np.asarray(xs, dtype=np.uint32)  # noqa: E731
    op = c["call"]
    if op in ("prefix_words", "first_words"):
        ctrs = c["ctrs"] if isinstance(c["ctrs"], int) else u32(c["ctrs"])
        if op == "prefix_words":
            got = bulk.prefix_words(c["alg"], u64(c["seeds"]), ctrs, c["nwords"], device="cpu")
        else:
            got = bulk.first_words(c["alg"], u64(c["seeds"]), ctrs, device="cpu")
        assert _sha32(got) == c["sha"]
    elif op == "source_stream_words":
        got = bulk.AlgorithmSource(c["alg"]).stream_words(c["seed"], c["ctr"], c["n"], device="cpu")
        assert _sha32(got) == c["sha"]
    elif op == "philox4x32":
        v = c["in"]
        assert _sha32(np.stack(bulk.philox4x32(*(u32(v[x]) for x in "abcdef")))) == c["sha"]
    elif op == "threefry4x32":
        v = c["in"]
        assert _sha32(np.stack(bulk.threefry4x32(*(u32(v[x]) for x in "abcdefgh")))) == c["sha"]
    elif op == "squares_keys":
        assert h16(np.asarray(bulk.squares_keys(u64(c["seeds"])), np.uint64).tobytes()) == c["sha"]
    elif op == "squares32":
        assert _sha32(bulk.squares32(u64(c["ctr"]), u64(c["key"]))) == c["sha"]
    elif op == "tyche_init":
        assert _sha32(np.stack(bulk.tyche_init(u64(c["seeds"]), u32(c["ctrs"])))) == c["sha"]
    elif op == "tyche_mix":
        v = c["in"]
        assert _sha32(np.stack(bulk.tyche_mix(*(u32(v[x]) for x in "abcd")))) == c["sha"]
    elif op == "tyche_advance_state":
        assert list(bulk.tyche_advance_state(tuple(c["state"]), c["steps"])) == c["res"]
    else:
        raise AssertionError(op)
