"""Mahalanobis depth, the rank study's parametric baseline (reference
univariate.py:49-152): (1 + (z - mu)' S^-1 (z - mu))^-1 with the
maximum-likelihood location/scatter.  d x d host algebra (one Cholesky
factorisation for all queries); it is not on the RRS hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import cho_factor, cho_solve

from .config import DimensionMismatch

SYMMETRY_TOL = 1e-10  # univariate.py:29


@dataclass(frozen=True)
class LocationScatter:
    """Location vector and symmetric positive-definite scatter matrix."""

    location: np.ndarray
    scatter: np.ndarray

    def __post_init__(self):
        loc = np.ascontiguousarray(self.location, dtype=np.float64).reshape(-1)
        sc = np.ascontiguousarray(self.scatter, dtype=np.float64)
        object.__setattr__(self, "location", loc)
        object.__setattr__(self, "scatter", sc)
        if sc.ndim != 2 or sc.shape != (loc.size, loc.size):
            raise ValueError("scatter must be square and match the location")
        if np.max(np.abs(sc - sc.T), initial=0.0) > SYMMETRY_TOL:
            raise ValueError("scatter not symmetric")
        try:
            np.linalg.cholesky(sc)
        except np.linalg.LinAlgError:
            raise ValueError("scatter not positive definite") from None


def estimate_mle(data) -> LocationScatter:
    """Column mean and the 1/n-normalised scatter."""
    x = data.x if hasattr(data, "x") else np.asarray(data, dtype=np.float64)
    if x.ndim != 2 or x.shape[0] <= 1:
        raise ValueError("need at least two observations to estimate scatter")
    mu = x.mean(axis=0)
    c = x - mu
    return LocationScatter(location=mu, scatter=c.T @ c / x.shape[0])


def _forms(Z: np.ndarray, est: LocationScatter) -> np.ndarray:
    if Z.shape[1] != est.location.size:
        raise DimensionMismatch(f"query dimension {Z.shape[1]} does not match location dimension "
                                f"{est.location.size}")
    diff = Z - est.location
    try:
        factor = cho_factor(est.scatter, lower=True)
    except np.linalg.LinAlgError:
        raise ValueError("scatter not positive definite") from None
    return (diff * cho_solve(factor, diff.T).T).sum(axis=1)


def mahalanobis_depth(z, est: LocationScatter) -> float:
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(1, -1)
    return float(1.0 / (1.0 + _forms(z, est)[0]))


def mahalanobis_depth_batch(queries, est: LocationScatter) -> np.ndarray:
    Z = np.atleast_2d(np.ascontiguousarray(queries, dtype=np.float64))
    return 1.0 / (1.0 + _forms(Z, est))
