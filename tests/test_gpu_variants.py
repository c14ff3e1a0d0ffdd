"""Every tuning variant of the fill kernels is bit-exact, not just the default.

The product library ships only the measured defaults. The alternatives
(Threefry round/injection/rotation pipe placement, CBRNG_TF_VARIANT; f32
conversion placement, CBRNG_CVT / CBRNG_CVT_MS; ILP, CBRNG_FILL_ILP; ...) live
in the tuning build (`make -C paper_2310_19925_b200/csrc tuning`,
-DCBRNG_TUNING=1), where environment knobs read once per process select them.
Each combination runs in a fresh child process bound to the tuning build and is
compared with the CPU oracle (the reference's algorithm, pinned to golden
vectors in test_oracle.py). Sizes cover full warp tiles, the remainder path and
a ragged tail. Skipped when the tuning build is absent: what ships is covered
by test_gpu_parity.py.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
TUNING_SO = ROOT / "paper_2310_19925_b200" / "_lib" / "libcbrng_b200_tuning.so"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not TUNING_SO.exists(), reason="tuning build absent (make -C csrc tuning)")]


CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from paper_2310_19925_b200 import _lib; _lib.use_tuning_build()
import paper_2310_19925_b200 as cb
from paper_2310_19925_b200 import bulk
from oracle import oracle as orc
bad = []
for alg in ("philox", "threefry", "squares"):
    for n in (4 * 32 * 16 * 3 + 4 * 37 + 3, 1 << 20):
        got = cb.uniform_f32_array(cb.make_generator(alg, 0xDEADBEEF1234, 7), n).cpu().numpy()
        ref = orc.words_to_f32(orc.stream_words(alg, 0xDEADBEEF1234, 7, n))
        if not np.array_equal(got, ref): bad.append(f"f32 {alg} {n}")
        w = cb.make_generator(alg, 99, 3).words(n).cpu().numpy()
        if not np.array_equal(w, orc.stream_words(alg, 99, 3, n)): bad.append(f"u32 {alg} {n}")
for alg in ("tyche", "threefry", "philox", "squares"):
    got = bulk.prefix_uniform_f32(alg, range(100, 100 + 777), 5, 52).cpu().numpy().reshape(-1)
    ref = orc.words_to_f32(orc.prefix_words_arange(alg, 100, 777, 5, 52))
    if not np.array_equal(got, ref): bad.append(f"prefix f32 {alg}")
print(json.dumps(bad))
"""


def _run(env_extra):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("cv", range(6))
def test_f32_conversion_variants(cv):
    assert _run({"CBRNG_CVT": str(cv), "CBRNG_CVT_MS": str(cv)}) == []


@pytest.mark.parametrize("v", range(9))
def test_threefry_variants(v):
    assert _run({"CBRNG_TF_VARIANT": str(v)}) == []


@pytest.mark.parametrize("inc", [0, 1, 2])
def test_squares_round1_forms(inc):
    """Squares round 1 as one 64-bit square per word (0) or by finite differences (1; 2: with every
    carry add forced onto the ALU pipe)."""
    assert _run({"CBRNG_SQ_INC": str(inc)}) == []


@pytest.mark.parametrize("ilp", [8, 12, 16])
def test_ilp_variants(ilp):
    assert _run({"CBRNG_FILL_ILP": str(ilp)}) == []


@pytest.mark.parametrize("ilp", [12, 16])
def test_squares_register_cap(ilp):
    """Squares fills capped at 6 CTAs/SM (<= 40 registers)."""
    assert _run({"CBRNG_SQ_MINB": "6", "CBRNG_FILL_ILP": str(ilp)}) == []


@pytest.mark.parametrize("ch", [4, 8])
def test_tyche_staging_width(ch):
    assert _run({"CBRNG_TY_CH": str(ch)}) == []


CHILD_ROWS256 = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from paper_2310_19925_b200 import _lib; _lib.use_tuning_build()
from paper_2310_19925_b200 import bulk
from oracle import oracle as orc
bad = []
for alg in ("philox", "threefry", "squares", "tyche"):
    for n in (5, 64, 1000):
        ref = orc.prefix_words_arange(alg, 9, n, 2, 256)
        if not np.array_equal(bulk.prefix_words(alg, range(9, 9 + n), 2, 256).cpu().numpy(), ref):
            bad.append(["u32", alg, n])
        got = bulk.prefix_uniform_f32(alg, range(9, 9 + n), 2, 256).cpu().numpy().reshape(-1)
        if not np.array_equal(got, orc.words_to_f32(ref)):
            bad.append(["f32", alg, n])
    seeds = np.arange(333, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    ctrs = np.arange(333, dtype=np.uint32) * np.uint32(7)
    got = bulk.prefix_words(alg, seeds, ctrs, 256).cpu().numpy()
    if not np.array_equal(got, orc.prefix_words(alg, seeds, ctrs, 256)):
        bad.append(["arrays", alg])
print(json.dumps(bad))
"""


@pytest.mark.parametrize("env", [{"CBRNG_MS_SPLIT": "0", "CBRNG_MS_TMA": "0"}, {"CBRNG_MS_SPLIT": "0", "CBRNG_MS_TMA": "1"},
                                 {"CBRNG_MS_SPLIT": "4"}, {"CBRNG_MS_SPLIT": "8"}, {"CBRNG_MS_SPLIT": "16"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_rows256_copy_out(env):
    """256-word rows through the staged kernel (LDS/STG or TMA-store copy-out) and the
    lanes-per-row kernel without staging (Philox / Threefry, 4 / 8 / 16 lanes per row)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CHILD_ROWS256 % str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert json.loads(r.stdout.strip().splitlines()[-1]) == []


CHILD_MISC = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from paper_2310_19925_b200 import _lib; _lib.use_tuning_build()
import paper_2310_19925_b200 as cb
from paper_2310_19925_b200 import bulk
from oracle import oracle as orc
bad = []
# Brownian, fused and per-step, from an odd start (chunked step table, wrapping counter)
for mode in ("fused", "per_step"):
    cfg = cb.SimConfig(300, 300, init_counter=0xFFFFFFA0, mode=mode)
    p = cb.init_particles(cfg)
    cb.brownian.run_steps(p, cfg, start_iteration=3)
    ref = orc.brownian_init("philox", 300, 0xFFFFFFA0)
    orc.brownian_steps("philox", ref, 3, 300, init_ctr=0xFFFFFFA0)
    for got, r in zip((p.x, p.y, p.vx, p.vy), ref):
        if not np.array_equal(got.cpu().numpy(), r): bad.append(["brownian", mode]); break
# grids: fills, Tyche rows, Box-Muller
for alg in ("philox", "threefry", "squares"):
    n = (1 << 20) + 9
    if not np.array_equal(cb.uniform_f32_array(cb.make_generator(alg, 5, 1), n).cpu().numpy(),
                          orc.words_to_f32(orc.stream_words(alg, 5, 1, n))): bad.append(["fill", alg])
got = bulk.prefix_uniform_f32("tyche", range(1000), 0, 256).cpu().numpy().reshape(-1)
if not np.array_equal(got, orc.words_to_f32(orc.prefix_words_arange("tyche", 0, 1000, 0, 256))): bad.append("tyche")
# Box-Muller: ragged sizes around the warp-specialised kernel's tiles, and
# 8-byte-aligned (not 16) outputs, which take the fused kernel
for n, off in ((4099, 0), (3, 0), (1 << 20, 0), (5 * 512 * 148 + 77, 0), (4099, 1)):
    z0 = torch.empty(n + off, dtype=torch.float64, device="cuda")[off:]
    z1 = torch.empty(n + off, dtype=torch.float64, device="cuda")[off:]
    cb.normal2_array(cb.make_generator("philox", 42, 0), n, out=(z0, z1))
    r0, r1 = orc.normal2("philox", 42, 0, n)
    for g, r in ((z0.cpu().numpy(), r0), (z1.cpu().numpy(), r1)):
        if not np.all(np.abs(g - r) <= 4 * np.spacing(np.maximum(np.abs(r), 1.0))): bad.append(["normal2", n, off])
print(json.dumps(bad))
"""


@pytest.mark.parametrize("env", [
    {"CBRNG_BROWNIAN_TAB": "0"}, {"CBRNG_BROWNIAN_TAB": "2"}, {"CBRNG_BROWNIAN_PINGPONG": "0"}, {"CBRNG_BROWNIAN_PDL": "0"},
    {"CBRNG_GRID_MULT": "0"}, {"CBRNG_GRID_MULT": "16"}, {"CBRNG_TY_GRID": "8"}, {"CBRNG_BM_GRID": "4"},
    *({"CBRNG_BM_LAYOUT": str(k)} for k in range(13)), *({"CBRNG_BM_SPLIT": str(k)} for k in range(1, 6)),
    {"CBRNG_BROWNIAN_SPLIT": "1"}, {"CBRNG_BROWNIAN_SPLIT": "2"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_misc_knobs(env):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-c", CHILD_MISC % str(ROOT)], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert json.loads(r.stdout.strip().splitlines()[-1]) == []
