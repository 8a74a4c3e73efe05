"""Filter-and-refine contraction (contract_tcf.cu): its halfspace counts are
bit-identical to the FFMA kernel's (contract.cu) for every direction, because
every pair whose FP16 one-product value is within the proven error bound is
recomputed with the FFMA kernel's own FP32 arithmetic.  Checked at the
config-4 shape, on tie-heavy integer data (exact zeros, duplicates: the
refinement queue overflows and the in-place path runs), at every d <= 64,
and end to end through RRS."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _counts(pkg, path, z, data, U):
    eng = pkg.engine()
    eng.set_contract_path(path)
    try:
        _, cle, cge = pkg.evaluate_directions_counts(z, data, U)
    finally:
        eng.set_contract_path("auto")
    return cle, cge


def _unit(rng, m, d):
    U = rng.standard_normal((m, d))
    return U / np.linalg.norm(U, axis=1)[:, None]


@pytest.mark.parametrize("dist", ["gaussian", "cauchy"])
def test_filter_equals_ffma_config4_shape(b200, dist):
    from paper_2506_08262_b200.synthetic import student_t, toeplitz_gaussian

    X = toeplitz_gaussian(50, 100_000, seed=0) if dist == "gaussian" else student_t(50, 100_000, 1.0, seed=0)
    rng = np.random.default_rng(21)
    data = b200.Dataset(X)
    U = _unit(rng, 1000, 50)
    # a cap of directions around one pole, like a late refinement (eps ~ 0.2 rad)
    pole = _unit(rng, 1, 50)[0]
    Ucap = b200.generate_batch(b200.CapSpec(b200.Pole(pole), 0.2), 1000, seed=3, refinement=12).directions
    for z in (X[3], 0.3 * X[7], np.zeros(50), X[11] + 1e-3 * rng.standard_normal(50), X[5] * 1e-6):
        for D in (U, Ucap):
            a = _counts(b200, "filter", z, data, D)
            f = _counts(b200, "ffma", z, data, D)
            assert np.array_equal(a[0], f[0]) and np.array_equal(a[1], f[1])


def test_filter_equals_ffma_tie_heavy(b200):
    rng = np.random.default_rng(5)
    X = rng.integers(-1, 2, size=(6000, 8)).astype(float)  # many duplicates and exact ties
    X[:500] = X[0]                                          # 500 copies of one point
    data = b200.Dataset(X)
    U = np.concatenate([np.eye(8), _unit(rng, 300, 8), np.ones((1, 8)) / np.sqrt(8)])
    for z in (X[0], X[700], np.zeros(8), np.full(8, 0.5)):
        a = _counts(b200, "filter", z, data, U)
        f = _counts(b200, "ffma", z, data, U)
        assert np.array_equal(a[0], f[0]) and np.array_equal(a[1], f[1])


@pytest.mark.parametrize("d", [1, 2, 5, 15, 16, 17, 31, 47, 48, 50, 63, 64])
def test_filter_all_dims(b200, d):
    rng = np.random.default_rng(d)
    n = 4096 + 77  # a partial last tile
    X = rng.standard_normal((n, d)) * rng.uniform(0.1, 10, d)
    data = b200.Dataset(X)
    U = _unit(rng, 300, d)  # a partial last direction block
    for z in (X[1], 0.5 * X[2], X[-1]):
        a = _counts(b200, "filter", z, data, U)
        f = _counts(b200, "ffma", z, data, U)
        assert np.array_equal(a[0], f[0]) and np.array_equal(a[1], f[1])


def test_filter_rrs_equals_ffma(b200):
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    X = toeplitz_gaussian(50, 20_000, seed=1)
    data = b200.Dataset(X)
    Z = np.concatenate([X[:40], 0.3 * X[40:80]])
    cfg = b200.RrsConfig(total_directions=4000, refinements=10, shrink=0.85, notion="halfspace", seed=2)
    eng = b200.engine()
    res = {}
    for path in ("filter", "ffma"):
        eng.set_contract_path(path)
        try:
            res[path] = b200.depth_batch_arrays(Z, data, cfg)
        finally:
            eng.set_contract_path("auto")
    for i in range(4):
        assert np.array_equal(res["filter"][i], res["ffma"][i])
