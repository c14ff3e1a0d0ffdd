"""Brownian-dynamics benchmark on sm_100a: drop-in for `cbrng.brownian`
(/root/reference/pkg/src/cbrng/brownian.py), the paper's macro-benchmark
(PAPER.md:100-139, :263).

Particles live in HBM as SoA float64 tensors; pid is implicit (pid_base + i,
the reference's np.arange layout, brownian.py:118) unless an explicit uint64
tensor is given. Each step re-derives the kick from stream (pid, init_counter +
it) inside the kernel: no RNG state, no random buffer.

`SimConfig.mode` picks the step kernel: "fused" (all steps in one launch, the
particle held in registers) or "per_step" (one launch per step, the paper's
kernel shape). Both produce bit-identical trajectories; `threads` is accepted
for API compatibility and ignored (the GPU grid replaces the thread pool).
"""

from __future__ import annotations

import dataclasses
import json
import math
import struct
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .generators import MASK32, Algorithm, as_algorithm

SNAPSHOT_MAGIC = b"CBRNSNP1"
_RECORD = struct.Struct("<Qdddd")  # pid, x, y, vx, vy (brownian.py:30)
_HEADER = struct.Struct("<8sQI")   # magic, n_particles, next_iteration (brownian.py:31)
FNV_OFFSET_BASIS = 0xCBF29CE484222325
MODES = {"per_step": _lib.BROWNIAN_PER_STEP, "fused": _lib.BROWNIAN_FUSED}


@dataclass
class SimConfig:
    """brownian.py:37-65, plus `mode` (kernel shape) and `device`."""

    n_particles: int
    steps: int
    dt: float = 0.01
    gamma: float = 0.1
    mass: float = 1.0
    threads: int = 1
    algorithm: Algorithm = Algorithm.PHILOX
    init_counter: int = 0
    mode: str = "fused"
    device: str | None = None

    def __post_init__(self):
        self.algorithm = as_algorithm(self.algorithm)
        if self.n_particles < 1:
            raise ValueError("n_particles must be >= 1")
        if self.steps < 0:
            raise ValueError("steps must be >= 0")
        if not self.dt >= 0:
            raise ValueError("dt must be non-negative")
        if self.gamma < 0:
            raise ValueError("gamma must be >= 0")
        if not self.mass > 0:
            raise ValueError("mass must be positive")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")


@dataclass
class Particles:
    """SoA particle store in HBM (brownian.py:68-88). `pid` is a uint64 tensor,
    or None for the implicit layout pid = pid_base + i."""

    pid: torch.Tensor | None
    x: torch.Tensor
    y: torch.Tensor
    vx: torch.Tensor
    vy: torch.Tensor
    pid_base: int = 0

    @property
    def n(self) -> int:
        return self.x.numel()

    def pid_array(self) -> np.ndarray:
        if self.pid is None:
            return np.arange(self.pid_base, self.pid_base + self.n, dtype=np.uint64)
        return self.pid.cpu().numpy()

    def copy(self) -> "Particles":
        return Particles(None if self.pid is None else self.pid.clone(), self.x.clone(), self.y.clone(),
                         self.vx.clone(), self.vy.clone(), self.pid_base)

    def host(self) -> dict[str, np.ndarray]:
        return {"pid": self.pid_array(), "x": self.x.cpu().numpy(), "y": self.y.cpu().numpy(),
                "vx": self.vx.cpu().numpy(), "vy": self.vy.cpu().numpy()}

    def _ptrs(self):
        return (_dev.ptr(self.pid), self.pid_base, self.x.data_ptr(), self.y.data_ptr(), self.vx.data_ptr(),
                self.vy.data_ptr())


@dataclass(frozen=True)
class TrajectoryChecksum:
    digest: int

    def __str__(self) -> str:
        return f"{self.digest:016x}"


@dataclass
class SimResult:
    particles: Particles
    checksum: TrajectoryChecksum | None
    wall_seconds: float
    particle_steps_per_second: float


def empty_particles(n: int, device=None, pid_base: int = 0) -> Particles:
    dev = _dev.cuda_device(device)
    mk = lambda: torch.empty(n, dtype=torch.float64, device=dev)  # noqa: E731
    return Particles(None, mk(), mk(), mk(), mk(), pid_base)


def init_particles(cfg: SimConfig, *, pid_base: int = 0, n: int | None = None) -> Particles:
    """8 words of stream (pid, init_counter) per particle (brownian.py:112-126).
    `pid_base`/`n` select a contiguous pid shard (multi-GPU)."""
    n = cfg.n_particles if n is None else n
    p = empty_particles(n, cfg.device, pid_base)
    pid_p, base, x, y, vx, vy = p._ptrs()
    _lib.check(_lib.lib().cbrng_brownian_init(int(cfg.algorithm), n, pid_p, base, cfg.init_counter & MASK32,
                                              x, y, vx, vy, _dev.sptr(p.x)), "brownian_init")
    return p


def _steps(p: Particles, cfg: SimConfig, first_it: int, nsteps: int, mode: str | None = None) -> None:
    pid_p, base, x, y, vx, vy = p._ptrs()
    _lib.check(_lib.lib().cbrng_brownian_steps(int(cfg.algorithm), p.n, pid_p, base, x, y, vx, vy,
                                               cfg.init_counter & MASK32, first_it, nsteps, cfg.gamma, cfg.mass,
                                               cfg.dt, MODES[mode or cfg.mode], _dev.sptr(p.x)), "brownian_steps")


def apply_forces_step(particles: Particles, iteration: int, cfg: SimConfig) -> Particles:
    """One dynamics step over all particles, in place (brownian.py:145-155)."""
    if iteration < 1:
        raise ValueError("iteration must be >= 1; counter 0 is reserved for init")
    _steps(particles, cfg, iteration, 1, "per_step")
    return particles


def run_steps(particles: Particles, cfg: SimConfig, start_iteration: int = 1, steps: int | None = None) -> Particles:
    """Advance `steps` (default cfg.steps) iterations from start_iteration, asynchronously."""
    if start_iteration < 1:
        raise ValueError("iteration must be >= 1; counter 0 is reserved for init")
    _steps(particles, cfg, start_iteration, cfg.steps if steps is None else steps)
    return particles


def run_sim(cfg: SimConfig, particles: Particles | None = None, start_iteration: int = 1,
            with_checksum: bool = True) -> SimResult:
    """brownian.py:164-195: init (unless given), cfg.steps steps, checksum.

    Wall time covers init + steps (as the reference's), measured with CUDA events.
    """
    dev = _dev.cuda_device(cfg.device)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host = time.perf_counter()
    e0.record(stream)
    if particles is None:
        particles = init_particles(cfg)
    if cfg.steps:
        run_steps(particles, cfg, start_iteration)
    e1.record(stream)
    e1.synchronize()
    wall = e0.elapsed_time(e1) / 1e3
    if wall <= 0:
        wall = time.perf_counter() - t_host
    digest = checksum(particles) if with_checksum else None
    rate = particles.n * cfg.steps / wall if wall > 0 else float("inf")
    return SimResult(particles, digest, wall, rate)


def _packed_records(particles: Particles) -> np.ndarray:
    """The pid-ordered `<Qdddd` records as host bytes: packed on the device from
    the SoA arrays (cbrng_pack_records), then one D2H copy into pinned memory."""
    n = particles.n
    rec = torch.empty(n * _RECORD.size, dtype=torch.uint8, device=particles.x.device)
    pid_p, base, x, y, vx, vy = particles._ptrs()
    _lib.check(_lib.lib().cbrng_pack_records(n, pid_p, base, x, y, vx, vy, rec.data_ptr(), _dev.sptr(particles.x)),
               "pack_records")
    h = torch.empty(rec.numel(), dtype=torch.uint8, pin_memory=True)
    h.copy_(rec, non_blocking=True)
    torch.cuda.current_stream(rec.device).synchronize()
    return h.numpy()


def checksum(particles: Particles) -> TrajectoryChecksum:
    """FNV-1a 64 over pid-ordered 40-byte records (brownian.py:209-223).

    FNV is byte-serial by definition (_kernels.py:89-96): the records are
    packed on the device, copied to the host and folded there by cbrng_fnv1a64.
    """
    if particles.pid is not None and particles.n > 1:
        bad = torch.zeros(1, dtype=torch.int32, device=particles.x.device)
        _lib.check(_lib.lib().cbrng_pid_order_check(particles.n, particles.pid.data_ptr(), bad.data_ptr(),
                                                    _dev.sptr(particles.x)), "pid_order_check")
        if int(bad.item()):
            raise ValueError("particles must be sorted by pid")
    if particles.n == 0:
        return TrajectoryChecksum(FNV_OFFSET_BASIS)
    rec = _packed_records(particles)
    return TrajectoryChecksum(int(_lib.lib().cbrng_fnv1a64(rec.ctypes.data, rec.size, FNV_OFFSET_BASIS)))


def stats(particles: Particles, acc: torch.Tensor | None = None) -> torch.Tensor:
    """Deterministic fixed-point moments + order-free digest (cbrng_brownian_stats),
    accumulated into `acc` (8 x int64 on the particles' device). Integer sums are
    associative, so shards reduced in any order (NCCL allreduce) give identical bits."""
    if acc is None:
        acc = torch.zeros(8, dtype=torch.int64, device=particles.x.device)
    pid_p, base, x, y, vx, vy = particles._ptrs()
    _lib.check(_lib.lib().cbrng_brownian_stats(particles.n, pid_p, base, x, y, vx, vy, acc.data_ptr(),
                                               _dev.sptr(particles.x)), "brownian_stats")
    return acc


def stats_summary(acc) -> dict:
    a = [int(v) for v in (acc.cpu().numpy() if isinstance(acc, torch.Tensor) else acc)]
    n = max(a[0], 1)
    return {"n": a[0], "mean_x": a[1] / 2**32 / n, "mean_y": a[2] / 2**32 / n, "mean_vx": a[3] / 2**32 / n,
            "mean_vy": a[4] / 2**32 / n, "mean_r2": a[5] / 2**24 / n, "mean_v2": a[6] / 2**24 / n,
            "digest": f"{a[7] & 0xFFFFFFFFFFFFFFFF:016x}"}


def save_snapshot(path, particles: Particles, next_iteration: int) -> None:
    """brownian.py:226-230"""
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(SNAPSHOT_MAGIC, particles.n, next_iteration))
        fh.write(_packed_records(particles).tobytes())


def load_snapshot(path, device=None) -> tuple[Particles, int]:
    """brownian.py:233-250"""
    with open(path, "rb") as fh:
        magic, n, next_iteration = _HEADER.unpack(fh.read(_HEADER.size))
        if magic != SNAPSHOT_MAGIC:
            raise ValueError("not a particle snapshot file")
        raw = np.frombuffer(fh.read(n * _RECORD.size), dtype=np.uint8)
    if raw.size != n * _RECORD.size:
        raise ValueError("truncated snapshot file")
    dev = _dev.cuda_device(device)
    rec = torch.from_numpy(raw.copy()).to(dev)
    pid = torch.empty(n, dtype=torch.uint64, device=dev)
    x, y, vx, vy = (torch.empty(n, dtype=torch.float64, device=dev) for _ in range(4))
    _lib.check(_lib.lib().cbrng_unpack_records(n, rec.data_ptr(), pid.data_ptr(), x.data_ptr(), y.data_ptr(),
                                               vx.data_ptr(), vy.data_ptr(), _dev.sptr(rec)), "unpack_records")
    return Particles(pid, x, y, vx, vy), next_iteration


def write_run_report(path, cfg: SimConfig, result: SimResult) -> None:
    """brownian.py:253-265"""
    payload = {
        "config": {**{k: v for k, v in dataclasses.asdict(cfg).items()}, "algorithm": cfg.algorithm.name.lower()},
        "checksum": str(result.checksum),
        "wall_seconds": result.wall_seconds,
        "particle_steps_per_second": result.particle_steps_per_second,
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh, indent=2)
        fh.write("\n")


def _slices(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous pid ranges (brownian.py:158-161); the multi-GPU shard map."""
    parts = max(1, min(parts, n))
    step = (n + parts - 1) // parts
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)]
