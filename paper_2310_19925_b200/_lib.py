"""ctypes binding of the sm_100a C ABI (include/cbrng_b200.h).

The product path has exactly one implementation: the CUDA kernels in
`_lib/libcbrng_b200.so`. There is no CPU fallback — if the library or a CUDA
device is missing, every generating call raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libcbrng_b200.so"
TUNING_LIB_PATH = LIB_DIR / "libcbrng_b200_tuning.so"  # `make -C csrc tuning`: tools/ sweeps only
CURAND_LIB_PATH = LIB_DIR / "libcbrng_curand_baseline.so"
CEILING_LIB_PATH = LIB_DIR / "libcbrng_ceiling.so"  # measurement only: HBM-free fills (bench.py)
HEADER = PKG.parent / "include" / "cbrng_b200.h"

CBRNG_OK, CBRNG_EINVAL, CBRNG_EALG, CBRNG_ECUDA, CBRNG_EALIGN = 0, -1, -2, -3, -4
BROWNIAN_PER_STEP, BROWNIAN_FUSED = 0, 1

_lock = threading.Lock()
_lib = None
_curand = None
_ceiling = None

u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p
u32, u64, i32, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_double

# name -> (restype, argtypes); mirrors include/cbrng_b200.h
SIGNATURES = {
    "cbrng_version": (C.c_char_p, []),
    "cbrng_last_error": (C.c_char_p, []),
    "cbrng_device_sm_count": (i32, [i32]),
    "cbrng_words": (i32, [i32, u64, u32, u64, vp, u64, vp, vp, vp]),
    "cbrng_uniform_f32": (i32, [i32, u64, u32, u64, vp, u64, vp, vp, vp]),
    "cbrng_uniform_f64": (i32, [i32, u64, u32, u64, vp, u64, vp, vp, vp]),
    "cbrng_normal2_f64": (i32, [i32, u64, u32, u64, vp, u64, vp, vp, vp, vp]),
    "cbrng_normal2_from_words": (i32, [vp, u64, vp, vp, vp]),
    "cbrng_words_multi": (i32, [i32, vp, vp, vp, vp, vp, vp, vp]),
    "cbrng_uniform_f32_multi": (i32, [i32, vp, vp, vp, vp, vp, vp, vp]),
    "cbrng_tyche_fill": (i32, [vp, u64, vp, vp]),
    "cbrng_prefix_words": (i32, [i32, vp, u64, vp, u32, u64, u32, vp, vp]),
    "cbrng_prefix_uniform_f32": (i32, [i32, vp, u64, vp, u32, u64, u32, vp, vp]),
    "cbrng_philox_block_lanes": (i32, [vp, vp, u64, u64, vp, vp]),
    "cbrng_philox4x32": (i32, [vp, vp, u64, vp, vp]),
    "cbrng_threefry4x32": (i32, [vp, vp, i32, u64, vp, vp]),
    "cbrng_squares32": (i32, [vp, vp, u64, vp, vp]),
    "cbrng_squares_keys": (i32, [vp, u64, vp, vp]),
    "cbrng_tyche_mix": (i32, [vp, u64, u32, vp]),
    "cbrng_tyche_init": (i32, [vp, u64, vp, u32, u64, vp, vp]),
    "cbrng_scalar": (i32, [i32, vp, u32, vp, u64]),
    "cbrng_brownian_init": (i32, [i32, u64, vp, u64, u32, vp, vp, vp, vp, vp]),
    "cbrng_brownian_steps": (i32, [i32, u64, vp, u64, vp, vp, vp, vp, u32, u64, u64, f64, f64, f64, i32, vp]),
    "cbrng_brownian_stats": (i32, [u64, vp, u64, vp, vp, vp, vp, vp, vp]),
    "cbrng_digest_u32": (i32, [vp, u64, u64, vp, vp]),
    "cbrng_pack_records": (i32, [u64, vp, u64, vp, vp, vp, vp, vp, vp]),
    "cbrng_unpack_records": (i32, [u64, vp, vp, vp, vp, vp, vp, vp]),
    "cbrng_pid_order_check": (i32, [u64, vp, vp, vp]),
    "cbrng_stream_byte_histogram": (i32, [i32, u64, u32, u64, vp, u64, vp, vp, vp]),
    "cbrng_prefix_byte_histogram": (i32, [i32, u64, u32, u32, u64, u32, vp, vp]),
    "cbrng_buffer_byte_histogram": (i32, [vp, u64, vp, vp]),
    "cbrng_avalanche": (i32, [i32, vp, vp, vp, u64, vp, vp]),
    "cbrng_pearson_partials": (i32, [vp, vp, u64, u32, vp, vp]),
    "cbrng_fnv1a64": (u64, [vp, u64, u64]),
}

CURAND_SIGNATURES = {
    "cbrng_curand_last_error": (C.c_char_p, []),
    "cbrng_curand_create": (vp, [u64, vp]),
    "cbrng_curand_destroy": (i32, [vp]),
    "cbrng_curand_set_offset": (i32, [vp, u64]),
    "cbrng_curand_u32": (i32, [vp, vp, u64]),
    "cbrng_curand_uniform_f32": (i32, [vp, vp, u64]),
    "cbrng_curand_uniform_f64": (i32, [vp, vp, u64]),
    "cbrng_curand_normal_f64": (i32, [vp, vp, u64]),
    "cbrng_curand_state_bytes": (u64, []),
    "cbrng_curand_brownian_init": (i32, [vp, u64, vp, vp, vp, vp, vp]),
    "cbrng_curand_brownian_steps": (i32, [vp, u64, vp, vp, vp, vp, u64, f64, f64, f64, i32, vp]),
    "cbrng_probe_store": (i32, [vp, u64, i32, i32, vp]),
    "cbrng_curand_rows": (i32, [u64, u64, u32, vp, vp]),
}


def build(force: bool = False) -> None:
    """Compile the CUDA libraries in-tree (make -C csrc); nvcc cross-compiles without a GPU."""
    cmd = ["make", "-s", "-j8", "-C", str(PKG / "csrc")]
    if force:
        subprocess.run(["make", "-s", "-C", str(PKG / "csrc"), "clean"], check=True)
    subprocess.run(cmd, check=True)


def build_tuning() -> None:
    """Compile libcbrng_b200_tuning.so (-DCBRNG_TUNING=1: CBRNG_* environment knobs and
    the alternative kernel variants) for tools/ sweeps and tests/test_gpu_variants.py."""
    subprocess.run(["make", "-s", "-j8", "-C", str(PKG / "csrc"), "tuning"], check=True)


def use_tuning_build() -> None:
    """Bind the tuning build instead of the product library (call before the first
    library call of the process; tools/ and tests/test_gpu_variants.py only)."""
    global LIB_PATH, _lib
    if _lib is not None and LIB_PATH != TUNING_LIB_PATH:
        raise RuntimeError("the product library is already bound in this process")
    LIB_PATH = TUNING_LIB_PATH


def _bind(path: Path, sigs: dict):
    L = C.CDLL(str(path))
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib():
    """The product library. Raises RuntimeError if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"CUDA library {LIB_PATH} is missing; run paper_2310_19925_b200._lib.build() "
                        "(there is no CPU fallback)")
                _lib = _bind(LIB_PATH, SIGNATURES)
    return _lib


def curand_lib():
    global _curand
    if _curand is None:
        with _lock:
            if _curand is None:
                _curand = _bind(CURAND_LIB_PATH, CURAND_SIGNATURES)
    return _curand


# cbrng_scalar ops (include/cbrng_b200.h)
(SCALAR_PHILOX_BLOCK, SCALAR_THREEFRY_BLOCK, SCALAR_SQUARES_KEY, SCALAR_SQUARES_ROUND, SCALAR_TYCHE_INIT,
 SCALAR_TYCHE_MIX, SCALAR_STREAM_WORDS, SCALAR_TYCHE_WORDS, SCALAR_TYCHE_SEED_WORDS) = range(9)
SCALAR_MAX_WORDS = 1 << 18
_scalar_tls = threading.local()


def scalar_small(op: int, args, nout: int) -> list:
    """cbrng_scalar for the block functions (ops 0-5, at most 4 result words): the
    same round trip into thread-local ctypes buffers, the words as a list."""
    tls = _scalar_tls
    buf = getattr(tls, "args", None)
    if buf is None:
        buf = tls.args = (C.c_uint64 * 16)()
    out = getattr(tls, "out", None)
    if out is None:
        out = tls.out = (C.c_uint32 * 4)()
    for i, a in enumerate(args):
        buf[i] = a & 0xFFFFFFFFFFFFFFFF
    check(lib().cbrng_scalar(op, buf, len(args), out, nout), "cbrng_scalar")
    return out[:nout]


def scalar(op: int, args, nout: int):
    """One synchronous scalar round trip through cbrng_scalar (host args, host
    result): a uint32 numpy array of nout words. Used by the reference's scalar
    API (block functions, generator windows); the GPU computes every word."""
    import numpy as np

    buf = getattr(_scalar_tls, "args", None)
    if buf is None:
        buf = _scalar_tls.args = (C.c_uint64 * 16)()
    for i, a in enumerate(args):
        buf[i] = int(a) & 0xFFFFFFFFFFFFFFFF
    out = np.empty(nout, np.uint32)
    check(lib().cbrng_scalar(op, buf, len(args), out.ctypes.data, nout), "cbrng_scalar")
    return out


def ceiling_lib():
    """The measurement-only build of the single-stream fills (-DCBRNG_CEILING=1): the same
    kernels with every store aimed at an L2-resident ring, so bench.py can time the
    HBM-free rate of the product's instruction stream. Never on a product path."""
    global _ceiling
    if _ceiling is None:
        with _lock:
            if _ceiling is None:
                _ceiling = _bind(CEILING_LIB_PATH, {k: SIGNATURES[k] for k in
                                                    ("cbrng_uniform_f32", "cbrng_normal2_f64", "cbrng_prefix_uniform_f32",
                                                     "cbrng_prefix_words", "cbrng_last_error")})
    return _ceiling


def last_error() -> str:
    msg = lib().cbrng_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map C-ABI status codes onto the reference's exception types."""
    if rc == CBRNG_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc in (CBRNG_EINVAL, CBRNG_EALG):
        raise ValueError(msg)
    raise RuntimeError(msg)


def require_cuda():
    """Fail loudly when no CUDA device is present (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2310_19925_b200 needs a CUDA device (B200); no CPU fallback exists")
    lib()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def header_symbols() -> list[str]:
    """Function names declared in include/cbrng_b200.h."""
    import re

    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(cbrng_[a-z0-9_]+)\s*\(", text, re.M)))
