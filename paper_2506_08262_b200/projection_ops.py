"""depthforge projection API on the device (projection.py:76-168).

The RRS path never materialises projections; these names exist for callers of
the reference's projection seam.  All three run ``proj64_kernel``
(csrc/api64.cu): FP64, acc = 0.0, ascending coordinate, separate multiply and
add -- the reference's proj_naive / proj_rect / proj_point_span arithmetic
(_kernels.pyx:120-199), so the scores are bit-identical to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import Dataset, DimensionMismatch, ParallelConfig


@dataclass(frozen=True)
class ProjectionMatrix:
    """m x n matrix of projection scores; row j projects all points onto u_j."""

    scores: np.ndarray

    @property
    def m(self) -> int:
        return self.scores.shape[0]

    @property
    def n(self) -> int:
        return self.scores.shape[1]


def _direction_matrix(dirs) -> np.ndarray:
    u = getattr(dirs, "directions", dirs)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.ndim != 2:
        raise DimensionMismatch("directions must form a 2-D matrix")
    return u


def _check_dims(d_data: int, d_dirs: int) -> None:
    if d_data != d_dirs:
        raise DimensionMismatch(f"direction dimension {d_dirs} does not match data dimension {d_data}")


def _project(x: np.ndarray, u: np.ndarray) -> np.ndarray:
    from .solver import _session

    with _session(None) as eng:
        return eng.project(x, u)


def project_naive(data: Dataset, dirs) -> ProjectionMatrix:
    """projection.py:99-105 (single-worker triple loop in the reference)."""
    u = _direction_matrix(dirs)
    _check_dims(data.dim, u.shape[1])
    return ProjectionMatrix(_project(data.x, u))


def project_parallel(data: Dataset, dirs, cfg: ParallelConfig | None = None) -> ProjectionMatrix:
    """projection.py:140-148; bit-identical to project_naive (cfg accepted, the
    device has no worker spans)."""
    u = _direction_matrix(dirs)
    _check_dims(data.dim, u.shape[1])
    return ProjectionMatrix(_project(data.x, u))


def project_point(z, dirs, cfg: ParallelConfig | None = None) -> np.ndarray:
    """projection.py:159-168: <z, u_j> for all directions, same arithmetic."""
    u = _direction_matrix(dirs)
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    _check_dims(z.size, u.shape[1])
    return _project(z.reshape(1, -1), u)[:, 0].copy()
