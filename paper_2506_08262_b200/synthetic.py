"""Synthetic inputs with the reference generators' exact bytes
(study/synthetic.py:21-96): Toeplitz Gaussian N(0, Sigma), Sigma_ij = 2^-|i-j|,
drawn from numpy's Philox bit generator keyed by the seed, and the elliptical
Student-t (nu = 1: heavy-tailed Cauchy) with the same scale matrix.  Used by
bench.py and the tests so the CPU and GPU legs see identical data.
"""

from __future__ import annotations

import numpy as np


def toeplitz_sigma(d: int) -> np.ndarray:
    idx = np.arange(d)
    return 2.0 ** (-np.abs(idx[:, None] - idx[None, :]))


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed % (1 << 64)))


def toeplitz_gaussian(dim: int, n: int, seed: int = 0) -> np.ndarray:
    if dim < 1 or n < 1:
        raise ValueError("dimension and sample size must be positive")
    chol = np.linalg.cholesky(toeplitz_sigma(dim))
    g = _rng(seed).standard_normal((n, dim))
    return g @ chol.T


def student_t(dim: int, n: int, nu: float, seed: int = 0) -> np.ndarray:
    if dim < 1 or n < 1:
        raise ValueError("dimension and sample size must be positive")
    if nu <= 0:
        raise ValueError("degrees of freedom must be positive")
    chol = np.linalg.cholesky(toeplitz_sigma(dim))
    rng = _rng(seed)
    g = rng.standard_normal((n, dim))
    w = rng.chisquare(nu, size=n)
    return (g @ chol.T) * np.sqrt(nu / w)[:, None]
