"""Device-buffer helpers shared by the host mirror of the reference API.

Outputs are torch tensors on the current CUDA device by default (the
B200-native placement: values stay in HBM for the next kernel). `device="cpu"`
returns a numpy array — the reference's own return type — via pinned host
memory; `out=` fills a caller buffer (CUDA tensor, pinned/pageable CPU tensor or
numpy array).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

NP_OF = {torch.uint32: np.uint32, torch.uint64: np.uint64, torch.float32: np.float32, torch.float64: np.float64,
         torch.int64: np.int64}
TORCH_OF = {np.dtype(v): k for k, v in NP_OF.items()}


def cuda_device(device=None) -> torch.device:
    _lib.require_cuda()
    if device is None or (isinstance(device, str) and device == "cuda"):
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"not a CUDA device: {device}")
    return d


def is_host(device) -> bool:
    return device is not None and torch.device(device).type == "cpu"


def empty(n, dtype, device=None) -> torch.Tensor:
    return torch.empty(n, dtype=dtype, device=cuda_device(device))


def ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def sptr(t: torch.Tensor | None = None) -> int:
    """Raw cudaStream_t of torch's current stream on the tensor's device."""
    if t is not None and t.is_cuda:
        return int(torch.cuda.current_stream(t.device).cuda_stream)
    return int(torch.cuda.current_stream().cuda_stream)


class Sink:
    """Where a fill lands: a device tensor the kernel writes, plus how to hand
    the result back (as-is, copied into a caller buffer, or to host numpy)."""

    def __init__(self, n, dtype: torch.dtype, out=None, device=None):
        self.n = n
        self.dtype = dtype
        self.user = out
        self.host = False
        if out is not None:
            if isinstance(out, np.ndarray):
                if out.dtype != np.dtype(NP_OF[dtype]) or out.size != n:
                    raise ValueError(f"out must be a {NP_OF[dtype].__name__}[{n}] array")
                self.host = True
                self.dev = empty(n, dtype)
            elif isinstance(out, torch.Tensor):
                if out.dtype != dtype or out.numel() != n:
                    raise ValueError(f"out must be a {dtype}[{n}] tensor")
                if out.is_cuda and out.is_contiguous() and out.data_ptr() % 16 == 0:
                    self.dev = out
                else:
                    self.host = not out.is_cuda
                    self.dev = empty(n, dtype, out.device if out.is_cuda else None)
            else:
                raise TypeError("out must be a torch.Tensor or numpy.ndarray")
        elif is_host(device):
            self.host = True
            self.dev = empty(n, dtype)
        else:
            self.dev = empty(n, dtype, device)

    def finish(self):
        if self.user is not None:
            if self.dev is self.user:
                return self.user
            if isinstance(self.user, np.ndarray):
                torch.from_numpy(self.user).copy_(self.dev)
                return self.user
            self.user.copy_(self.dev.view(self.user.shape))
            return self.user
        if self.host:
            h = torch.empty(self.n, dtype=self.dtype, pin_memory=True)
            h.copy_(self.dev, non_blocking=True)
            torch.cuda.current_stream(self.dev.device).synchronize()
            return h.numpy()
        return self.dev


HOST_CHUNK_BYTES = 64 << 20  # chunk of a pipelined device -> host fill


def pinned_host_target(out, n: int, dtype: torch.dtype, device) -> torch.Tensor | None:
    """The pinned host tensor a fill of n elements can stream into chunk by chunk,
    or None when the destination is not host memory that can take async copies
    (device outputs, numpy / pageable buffers, small fills keep the one-shot path)."""
    if n * torch.empty(0, dtype=dtype).element_size() < 2 * HOST_CHUNK_BYTES:
        return None
    if out is None:
        return torch.empty(n, dtype=dtype, pin_memory=True) if is_host(device) else None
    if (isinstance(out, torch.Tensor) and not out.is_cuda and out.is_pinned() and out.is_contiguous()
            and out.dtype == dtype and out.numel() == n):
        return out.view(-1)
    return None


def pipelined_host_fill(n: int, dtype: torch.dtype, hosts: list, launch, row: int = 1) -> None:
    """Fill host tensors `hosts` (pinned, n*row elements each) by generating
    HOST_CHUNK_BYTES chunks into two alternating device buffers per output and
    copying each to the host on a second stream while the next chunk is
    generated. Chunked copies also reach ~56 GB/s where one multi-GiB copy
    gets ~53 (tools/probes/probe_d2h.py). launch(dev_ptrs, first, count,
    stream_ptr) generates elements [first, first + count) (rows of `row`)."""
    dev = cuda_device()
    esz = torch.empty(0, dtype=dtype).element_size()
    k = max(1, HOST_CHUNK_BYTES // (esz * row))
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    bufs = [[torch.empty(k * row, dtype=dtype, device=dev) for _ in hosts] for _ in range(2)]
    copied = [None, None]
    try:
        for i, off in enumerate(range(0, n, k)):
            slot, m = i & 1, min(k, n - off)
            if copied[slot] is not None:
                comp.wait_event(copied[slot])  # the slot's previous chunk has left the GPU
            launch([b.data_ptr() for b in bufs[slot]], off, m, int(comp.cuda_stream))
            ready = torch.cuda.Event()
            ready.record(comp)
            copy.wait_event(ready)
            with torch.cuda.stream(copy):
                for h, b in zip(hosts, bufs[slot]):
                    h[off * row:(off + m) * row].copy_(b[:m * row], non_blocking=True)
            done = torch.cuda.Event()
            done.record(copy)
            copied[slot] = done
    finally:
        # also on error: no copy may still read a device buffer once it is freed
        copy.synchronize()


def to_numpy(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def as_dev(x, np_dtype, device=None) -> torch.Tensor:
    """Contiguous CUDA tensor of dtype np_dtype from numpy / python / torch input."""
    tdt = TORCH_OF[np.dtype(np_dtype)]
    if isinstance(x, torch.Tensor):
        dev = cuda_device(device if device is not None else (x.device if x.is_cuda else None))
        if x.dtype != tdt:
            same_width_ints = (not x.dtype.is_floating_point and not tdt.is_floating_point
                               and x.element_size() == np.dtype(np_dtype).itemsize)
            if same_width_ints:
                x = x.contiguous().view(tdt)  # two's-complement reinterpretation, as numpy's astype
            elif x.dtype.is_floating_point and tdt.is_floating_point:
                x = x.to(tdt)
            else:  # integer width changes: numpy's wrapping conversion on the host
                x = torch.from_numpy(np.ascontiguousarray(x.detach().cpu().numpy().astype(np_dtype)))
        return x.to(dev).contiguous()
    a = np.ascontiguousarray(np.asarray(x).astype(np_dtype, copy=False))
    return torch.from_numpy(a).to(cuda_device(device))
