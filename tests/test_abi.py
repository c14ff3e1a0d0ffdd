"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/cbrng_b200.h declares, and host-only entry points behave
(no GPU compute here)."""

from __future__ import annotations

import ctypes
import subprocess

import pytest

from paper_2310_19925_b200 import _lib


def test_library_loads_and_versions():
    L = _lib.lib()
    assert L.cbrng_version().startswith(b"cbrng-b200")


def test_header_symbols_exported():
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(_lib.SIGNATURES) == declared  # the ctypes table mirrors the header exactly


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_fnv_host_entry_point(golden):
    L = _lib.lib()
    buf = (ctypes.c_uint8 * 40)()
    assert L.cbrng_fnv1a64(ctypes.addressof(buf), 40, 0xCBF29CE484222325) == golden["fnv"]["zero40"]
    data = bytes(range(256)) * 3
    b = ctypes.create_string_buffer(data, len(data))
    assert L.cbrng_fnv1a64(ctypes.addressof(b), len(data), 0xCBF29CE484222325) == golden["fnv"]["bytes0_255x3"]


def test_unknown_algorithm_is_rejected_before_launch():
    L = _lib.lib()
    rc = L.cbrng_words(9, 0, 0, 0, None, 16, None, None, None)
    assert rc == _lib.CBRNG_EALG
    assert b"unknown algorithm" in L.cbrng_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_invalid_brownian_arguments_are_rejected():
    L = _lib.lib()
    rc = L.cbrng_brownian_steps(0, 4, None, 0, None, None, None, None, 0, 0, 1, 0.1, 1.0, 0.01, 1, None)
    assert rc == _lib.CBRNG_EINVAL and b"iteration" in L.cbrng_last_error()
    rc = L.cbrng_brownian_steps(0, 4, None, 0, None, None, None, None, 0, 1, 1, 0.1, 1.0, 0.01, 7, None)
    assert rc == _lib.CBRNG_EINVAL


def test_generating_without_cuda_fails_loudly():
    import torch

    import paper_2310_19925_b200 as cb

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cb.make_generator("philox", 42, 0).words(16)


def test_curand_baseline_is_a_separate_library():
    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "curand" not in out
    assert _lib.CURAND_LIB_PATH.exists()
