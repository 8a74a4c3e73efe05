"""depthforge univariate API on the device (univariate.py:33-107, 155-184).

``depth_of_projections`` runs ``span_depth64_kernel`` (csrc/api64.cu) over the
caller's px / pz: exact FP64 order statistics (radix select on 64-bit keys),
the reference's median rule and deviation arithmetic (_kernels.pyx:202-351),
so the depths are bit-identical to the reference's span kernels.  The scalar
1-D forms are the m = 1 case of the same kernel (the reference documents the
scalar forms and the batch spans as agreeing bit for bit, univariate.py:3-4).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import NOTIONS


@dataclass(frozen=True)
class ProjectedSample:
    """Projection scores of the dataset (values) and of the query point."""

    values: np.ndarray
    query: float

    def __post_init__(self):
        values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "query", float(self.query))
        if values.size < 1:
            raise ValueError("empty projection")
        if not (np.isfinite(values).all() and np.isfinite(self.query)):
            raise ValueError("projected sample contains non-finite entries")


def depth_of_projections(notion: str, px: np.ndarray, pz: np.ndarray, out: np.ndarray | None = None, *,
                         workers: int = 1, block_size: int = 256) -> np.ndarray:
    """univariate.py:162-184: depth of pz[j] within px[j, :] for every j
    (workers / block_size accepted for API parity)."""
    from .solver import _session

    if notion not in NOTIONS:
        raise ValueError(f"unknown depth notion {notion!r}")
    px = np.ascontiguousarray(px, dtype=np.float64)
    pz = np.ascontiguousarray(pz, dtype=np.float64).reshape(-1)
    if px.ndim != 2 or px.shape[1] < 1:
        raise ValueError("empty projection")
    if pz.size != px.shape[0]:
        raise ValueError("pz must hold one query score per direction")
    res = np.empty(px.shape[0]) if out is None or not out.flags.c_contiguous else out
    with _session(None) as eng:
        eng.depth_of_projections(notion, px, pz, res)
    if out is not None and res is not out:
        out[...] = res
        return out
    return res


def _one(notion: str, s: ProjectedSample) -> float:
    return float(depth_of_projections(notion, s.values[None, :], np.array([s.query]))[0])


def halfspace_depth_1d(s: ProjectedSample) -> float:
    """min(#{values <= query}, #{values >= query}) / n, ties on both sides."""
    return _one("halfspace", s)


def projection_depth_1d(s: ProjectedSample) -> float:
    """(1 + |query - med| / MAD)^-1; MAD = 0 gives 1 at the median, else 0."""
    return _one("projection", s)


def asym_projection_depth_1d(s: ProjectedSample) -> float:
    """(1 + (query - med)+ / MAD+)^-1; 1 whenever the query is at or below med."""
    return _one("asym_projection", s)
