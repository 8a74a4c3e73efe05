"""Reference-facing types of the RRS hot path, same names, fields, defaults and
validation messages as depthforge (paths relative to
/root/reference/pkg/src/depthforge):

  DimensionMismatch   projection.py:23-24
  ParallelConfig      projection.py:27-41   (accepted for API parity; the
                                             device path has no worker spans)
  Dataset             projection.py:44-75
  RrsConfig           optimizer.py:42-66
  RefinementRecord    optimizer.py:69-75
  DepthResult         optimizer.py:78-83
  PhaseTimer          optimizer.py:86-95
  Pole / CapSpec / DirectionBatch / SubStream   directions.py:37-94
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np

NOTIONS = ("halfspace", "projection", "asym_projection")  # univariate.py:27
POLE_UPDATE_MODES = ("per_refinement", "per_direction")  # optimizer.py:39
HALF_PI = math.pi / 2.0  # optimizer.py:37
UNIT_NORM_TOL = 1e-12  # directions.py:32


class DimensionMismatch(ValueError):
    """Operands disagree on the space dimension or shape."""


def _default_workers() -> int:
    env = os.environ.get("DEPTHFORGE_WORKERS")
    if env:
        try:
            v = int(env)
            if v >= 1:
                return v
        except ValueError:
            pass
    return os.cpu_count() or 1


@dataclass(frozen=True)
class ParallelConfig:
    workers: int = field(default_factory=_default_workers)
    block_size: int = 256
    d_chunk: int = 256

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.d_chunk < 1:
            raise ValueError("d_chunk must be >= 1")


def _all_finite(x: np.ndarray) -> bool:
    """np.isfinite(x).all(); large matrices use multi-threaded max / min
    reductions (NaN propagates through both, +-inf shows up in one)."""
    if x.size < (1 << 22):
        return bool(np.isfinite(x).all())
    try:
        import torch
    except ImportError:  # pragma: no cover
        return bool(np.isfinite(x).all())
    t = torch.from_numpy(x)
    return bool(torch.isfinite(t.amax())) and bool(torch.isfinite(t.amin()))


class Dataset:
    """An n x d row-major matrix of observations (64-bit floats, all finite)."""

    def __init__(self, rows):
        x = np.ascontiguousarray(rows, dtype=np.float64)
        if x.ndim == 1:
            x = x.reshape(1, -1)
        if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] < 1:
            raise ValueError("dataset must be a non-empty 2-D matrix")
        if not _all_finite(x):
            raise ValueError("dataset contains non-finite entries")
        self.x = x
        self._xt = None
        self._token = object()  # identity of the device-resident copy

    @property
    def n(self) -> int:
        return self.x.shape[0]

    @property
    def dim(self) -> int:
        return self.x.shape[1]

    @property
    def xt(self) -> np.ndarray:
        if self._xt is None:
            self._xt = np.ascontiguousarray(self.x.T)
        return self._xt

    def __repr__(self):
        return f"Dataset(n={self.n}, dim={self.dim})"


@dataclass(frozen=True)
class RrsConfig:
    """Search budget: k = total_directions (NRandom), r = refinements
    (n_refinements), alpha = shrink (sphcap_shrink)."""

    total_directions: int = 100_000
    refinements: int = 40
    shrink: float = 0.9
    notion: str = "projection"
    seed: int = 0
    parallel: ParallelConfig = field(default_factory=ParallelConfig)
    pole_update: str = "per_refinement"
    # B200 extension (halfspace): stop a query once its best count equals the
    # number of data rows coinciding with it -- the strict-< update
    # (optimizer.py:202) can then never fire again, so depth, argmin and trace
    # are bitwise those of the full run; off by default (the reference's cost)
    early_exit: bool = False

    def __post_init__(self):
        if self.refinements < 1 or self.total_directions < self.refinements:
            raise ValueError("need total_directions >= refinements >= 1")
        if not (0.0 < self.shrink < 1.0):
            raise ValueError("shrink factor must lie in (0, 1)")
        if self.notion not in NOTIONS:
            raise ValueError(f"unknown depth notion {self.notion!r}")
        if self.pole_update not in POLE_UPDATE_MODES:
            raise ValueError(f"unknown pole update mode {self.pole_update!r}")

    @property
    def directions_per_refinement(self) -> int:
        return -(-self.total_directions // self.refinements)

    def epsilons(self) -> list[float]:
        """optimizer.py:175, evaluated in Python exactly like the reference."""
        return [HALF_PI * self.shrink**l for l in range(self.refinements)]


@dataclass(frozen=True)
class RefinementRecord:
    best_depth: float
    epsilon: float
    pole: np.ndarray


@dataclass(frozen=True)
class DepthResult:
    depth: float
    argmin_direction: np.ndarray
    trace: tuple[RefinementRecord, ...]
    directions_used: int


class PhaseTimer:
    """Accumulates time per phase (generation/projection/univariate).  On the
    device path the numbers are CUDA-event times of the stage kernels."""

    def __init__(self):
        self.seconds = {"generation": 0.0, "projection": 0.0, "univariate": 0.0}
        self._lock = threading.Lock()

    def add(self, phase: str, dt: float) -> None:
        with self._lock:
            self.seconds[phase] += dt


@dataclass(frozen=True)
class Pole:
    p: np.ndarray

    def __post_init__(self):
        p = np.ascontiguousarray(self.p, dtype=np.float64).reshape(-1)
        object.__setattr__(self, "p", p)
        if abs(float(np.linalg.norm(p)) - 1.0) > UNIT_NORM_TOL:
            raise ValueError("pole must have unit norm")


@dataclass(frozen=True)
class CapSpec:
    pole: Pole
    epsilon: float

    def __post_init__(self):
        if not (0.0 < self.epsilon <= math.pi / 2 + 1e-15):
            raise ValueError("cap half-angle must lie in (0, pi/2]")


@dataclass(frozen=True)
class DirectionBatch:
    directions: np.ndarray
    seed_info: tuple[int, int]

    @property
    def m(self) -> int:
        return self.directions.shape[0]

    @property
    def dim(self) -> int:
        return self.directions.shape[1]
