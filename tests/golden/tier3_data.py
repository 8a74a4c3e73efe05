"""Machine-independent synthetic data for the full-shape tier-3 fixtures.

The reference generators (study/synthetic.py:83-96) compute ``g @ chol(Sigma).T``
with BLAS, whose bytes depend on the CPU kernel OpenBLAS picks; a fixture made
here could then describe a dataset the GPU box regenerates differently.  For
Sigma_ij = 2^-|i-j| the Cholesky factor is the AR(1) filter
``x_0 = g_0, x_l = x_{l-1}/2 + sqrt(3/4) g_l``, which is evaluated here with
elementwise numpy ops only (IEEE, no contraction), so the bytes are the same on
every x86-64 box.  Same distribution as the reference generator (N(0, Sigma);
the elliptical Student-t scales rows by sqrt(nu/w), w ~ chi2(nu), drawn from
the same Philox stream after the normals, like gen_student_t).

Shared by tests/golden/make_tier3.py (which runs the real reference on these
arrays) and tests/test_tier3_full_shapes.py (which runs the CUDA path on them).
"""

from __future__ import annotations

import hashlib

import numpy as np

_S = np.sqrt(0.75)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed % (1 << 64)))


def _ar1(g: np.ndarray) -> np.ndarray:
    x = np.empty_like(g)
    x[:, 0] = g[:, 0]
    for l in range(1, g.shape[1]):
        np.add(x[:, l - 1] * 0.5, g[:, l] * _S, out=x[:, l])
    return x


def gaussian(d: int, n: int, seed: int) -> np.ndarray:
    return _ar1(_rng(seed).standard_normal((n, d)))


def cauchy(d: int, n: int, seed: int) -> np.ndarray:
    rng = _rng(seed)
    g = rng.standard_normal((n, d))
    w = rng.chisquare(1.0, size=n)
    return _ar1(g) * np.sqrt(1.0 / w)[:, None]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def subset(n: int, count: int, seed: int = 3) -> np.ndarray:
    """Fixed random query subset (np.random.Philox(key=3))."""
    return np.sort(_rng(seed).choice(n, size=count, replace=False))


# (tag, notion, n, d, dist, k, r, alpha) -- BASELINE.json configs 2-5
CASES = {
    "c2": ("projection", 10_000, 20, "gauss", 20_000, 20, 0.9),
    "c3": ("asym_projection", 50_000, 50, "cauchy", 20_000, 20, 0.9),
    "c4": ("halfspace", 100_000, 50, "gauss", 20_000, 20, 0.9),
    "c5h": ("halfspace", 1_000_000, 200, "gauss", 20_000, 20, 0.9),
    "c5p": ("projection", 1_000_000, 200, "gauss", 20_000, 20, 0.9),
}


def dataset(tag: str) -> np.ndarray:
    notion, n, d, dist, *_ = CASES[tag]
    return gaussian(d, n, 0) if dist == "gauss" else cauchy(d, n, 0)


def queries(tag: str, X: np.ndarray) -> np.ndarray:
    """Query sets: config 4 off-sample (0.3 x_i and a fresh seed-2 sample, SURVEY
    §8(d): in-sample depths are all 1/n there) plus a few in-sample rows;
    configs 2/3 in-sample rows (the all-points workload); config 5 a mix."""
    n, d = X.shape
    if tag == "c2":
        return X[subset(n, 64)]
    if tag == "c3":
        return X[subset(n, 32)]
    # (a fresh sample at full scale lies outside the hull of n points in d = 50
    # or 200 -- depth 0 -- so the fresh seed-2 sample is shrunk toward the centre)
    if tag == "c4":
        idx = subset(n, 40)
        return np.concatenate([0.3 * X[idx[:32]], 0.15 * gaussian(d, 32, 2), X[idx[32:]]])
    if tag in ("c5h", "c5p"):
        idx = subset(n, 4)
        return np.concatenate([X[idx[:2]], 0.3 * X[idx[2:]], 0.1 * gaussian(d, 2, 2)])
    raise KeyError(tag)
