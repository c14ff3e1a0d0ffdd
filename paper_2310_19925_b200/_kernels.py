"""Drop-in for the reference's numba kernels (`cbrng._kernels`, _kernels.py:1-96)
on the C ABI: same names, same in-place conventions, numpy in / numpy out.

  tyche_fill(state, out)                       -> cbrng_tyche_fill (serial chain, one GPU thread)
  philox_block_lanes(seeds, scs, block, out)   -> cbrng_philox_block_lanes
  fnv1a64(data)                                -> cbrng_fnv1a64 (byte-serial, host)
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib

FNV_OFFSET_BASIS = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def tyche_fill(state: np.ndarray, out: np.ndarray) -> None:
    """_kernels.py:22-44: fill `out` with len(out) Tyche words, update `state` in place."""
    st = np.ascontiguousarray(state, dtype=np.uint64)
    n = int(out.shape[0])
    dev = _dev.empty(max(n, 1), torch.uint32)
    _lib.check(_lib.lib().cbrng_tyche_fill(st.ctypes.data, n, dev.data_ptr(), _dev.sptr(dev)), "tyche_fill")
    if n:
        out[...] = dev[:n].cpu().numpy()
    state[...] = st


def philox_block_lanes(seeds: np.ndarray, stream_ctrs: np.ndarray, block_ctr: int, out: np.ndarray) -> None:
    """_kernels.py:54-86: out[i, :] = Philox block `block_ctr` of stream (seeds[i], stream_ctrs[i])."""
    from . import bulk

    out[...] = bulk.philox_block_lanes(seeds, stream_ctrs, int(block_ctr), device="cpu")


def fnv1a64(data: np.ndarray) -> int:
    """_kernels.py:89-96"""
    b = np.ascontiguousarray(data, dtype=np.uint8)
    return int(_lib.lib().cbrng_fnv1a64(b.ctypes.data, b.size, FNV_OFFSET_BASIS))
