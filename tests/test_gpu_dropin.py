"""The drop-in: reference test cases run through ``import paper_2506_08262_b200
as depthforge`` on the B200.

Ported (restated, same cases and expectations) from the reference's own
suite: tests/test_univariate.py, test_projection.py, test_philox_directions.py
and test_optimizer.py (paths under /root/reference/pkg).  Where the
reference's expectation is "bit-identical to the reference core", the checker
is the golden fixture made by the real reference (tests/golden/golden.npz) or
the pinned CPU oracle (oracle/).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def depthforge(b200):
    import paper_2506_08262_b200 as depthforge

    return depthforge


def S(df, values, query):
    return df.ProjectedSample(values=np.asarray(values, dtype=float), query=query)


# ------------------------------------------------ test_univariate.py cases --
def test_halfspace_hand_cases(depthforge):
    df = depthforge
    assert df.halfspace_depth_1d(S(df, [1, 2, 3, 4, 5], 3)) == 3 / 5
    assert df.halfspace_depth_1d(S(df, [1, 2, 3], 0)) == 0.0
    assert df.halfspace_depth_1d(S(df, [1, 1, 2], 1)) == 2 / 3
    with pytest.raises(ValueError, match="empty projection"):
        df.ProjectedSample(values=np.array([]), query=0.0)


def test_halfspace_zero_iff_outside_and_counting_oracle(depthforge):
    df = depthforge
    rng = np.random.default_rng(0)
    for _ in range(60):
        v = rng.standard_normal(rng.integers(1, 20))
        q = rng.standard_normal() * 2
        assert (df.halfspace_depth_1d(S(df, v, q)) == 0.0) == (q < v.min() or q > v.max())
    rng = np.random.default_rng(1)
    for _ in range(60):
        v = rng.integers(-5, 6, size=rng.integers(1, 30)).astype(float)
        q = float(rng.integers(-6, 7))
        want = min(np.count_nonzero(v <= q), np.count_nonzero(v >= q)) / v.size
        assert df.halfspace_depth_1d(S(df, v, q)) == want


def test_projection_depth_hand_cases(depthforge):
    df = depthforge
    assert df.projection_depth_1d(S(df, [1, 2, 3, 4, 7], 3)) == 1.0
    assert df.projection_depth_1d(S(df, [1, 2, 3, 4, 5], 5)) == pytest.approx(1 / 3, rel=1e-15)
    assert df.projection_depth_1d(S(df, [1, 2, 3, 4, 5], 4)) == pytest.approx(1 / 2, rel=1e-15)
    assert df.projection_depth_1d(S(df, [2, 2, 2], 2)) == 1.0
    assert df.projection_depth_1d(S(df, [2, 2, 2], 3)) == 0.0
    v = np.array([0.0, 1.0, 2.0, 5.0, 9.0])
    depths = [df.projection_depth_1d(S(df, v, q)) for q in np.linspace(2, 30, 40)]
    assert all(a >= b for a, b in zip(depths, depths[1:]))


def test_asym_projection_hand_cases(depthforge):
    df = depthforge
    assert df.asym_projection_depth_1d(S(df, [1, 2, 3, 4, 5], 2)) == 1.0
    assert df.asym_projection_depth_1d(S(df, [1, 2, 3, 4, 5], 3)) == 1.0
    assert df.asym_projection_depth_1d(S(df, [1, 2, 3, 4, 5], 5)) == pytest.approx(3 / 7, rel=1e-15)
    assert df.asym_projection_depth_1d(S(df, [1.0, 1.0, 1.0], 0.5)) == 1.0
    assert df.asym_projection_depth_1d(S(df, [1.0, 1.0, 1.0], 2.0)) == 0.0


def _sort_median(v):
    s = np.sort(v)
    n = s.size
    return s[n // 2] if n % 2 else (s[n // 2 - 1] + s[n // 2]) / 2.0


def test_projection_depths_match_sort_oracle(depthforge):
    """test_univariate.py:93-127 (sort oracle, rel 1e-12), batched through
    depth_of_projections and checked per row through the scalar forms too."""
    df = depthforge
    rng = np.random.default_rng(7)
    for _ in range(40):
        n = int(rng.integers(1, 41))
        v = np.round(rng.uniform(-1e6, 1e6, n), int(rng.integers(0, 3)))
        q = float(np.round(rng.uniform(-1e6, 1e6), 1))
        med = _sort_median(v)
        mad = _sort_median(np.abs(v - med))
        dev = abs(q - med)
        want_p = (1.0 if dev == 0 else 0.0) if mad == 0 else 1.0 / (1.0 + dev / mad)
        pos = (v - med)[(v - med) > 0]
        want_a = 1.0 if q - med <= 0 else (0.0 if pos.size == 0 else 1.0 / (1.0 + (q - med) / _sort_median(pos)))
        assert df.projection_depth_1d(S(df, v, q)) == pytest.approx(want_p, rel=1e-12, abs=0.0)
        assert df.asym_projection_depth_1d(S(df, v, q)) == pytest.approx(want_a, rel=1e-12, abs=0.0)
        # antipodal symmetry of the symmetric notions (test_univariate.py:139-160)
        assert df.halfspace_depth_1d(S(df, v, q)) == df.halfspace_depth_1d(S(df, -v, -q))
        assert df.projection_depth_1d(S(df, v, q)) == df.projection_depth_1d(S(df, -v, -q))


def test_depth_of_projections_bitexact_vs_reference_spans(depthforge, golden):
    """The reference's span kernels on tie-heavy rows (make_golden.py), every
    notion and n in {1, 2, 3, 18, 101, 1024}: bit-identical depths."""
    df = depthforge
    for n in (1, 2, 3, 18, 101, 1024):
        px, pz = golden[f"span_n{n}_px"], golden[f"span_n{n}_pz"]
        for notion in ("halfspace", "projection", "asym_projection"):
            got = df.depth_of_projections(notion, px, pz)
            assert np.array_equal(got, golden[f"span_n{n}_{notion}"]), (n, notion)
            # batch equals scalar (test_univariate.py:190-204)
            one = getattr(df, f"{notion}_depth_1d")
            for j in (0, 17, 59):
                assert one(df.ProjectedSample(px[j], pz[j])) == got[j]
    for notion in ("halfspace", "projection", "asym_projection"):
        out = np.empty(3)
        df.depth_of_projections(notion, golden["degen_px"], golden["degen_pz"], out)
        assert np.array_equal(out, golden[f"degen_{notion}"])
    with pytest.raises(ValueError, match="unknown depth notion"):
        df.depth_of_projections("tukey", golden["degen_px"], golden["degen_pz"])


def test_depth_range_bounds(depthforge):
    df = depthforge
    rng = np.random.default_rng(3)
    px = rng.standard_cauchy((64, 257))
    pz = rng.standard_cauchy(64) * 3
    for notion in ("halfspace", "projection", "asym_projection"):
        d = df.depth_of_projections(notion, px, pz)
        assert np.all((d >= 0.0) & (d <= 1.0))


# ------------------------------------------------ test_projection.py cases --
def test_projection_cases(depthforge, golden, orc):
    df = depthforge
    rng = np.random.default_rng(4)
    x = rng.standard_normal((9, 4))
    data = df.Dataset(x)
    assert np.array_equal(df.project_parallel(data, np.eye(4)).scores, x.T)
    e1 = np.zeros((1, 4))
    e1[0, 0] = 1.0
    assert np.array_equal(df.project_naive(data, e1).scores[0], x[:, 0])
    # the reference's proj_naive on random data: bit-identical
    got = df.project_naive(df.Dataset(golden["proj_x"]), golden["proj_u"]).scores
    assert np.array_equal(got, golden["proj_out"])
    with pytest.raises(df.DimensionMismatch):
        df.project_parallel(data, np.ones((2, 3)))
    # randomized shapes, bit-exact against the pinned oracle's FP64 no-FMA product
    for n, d, m in [(1, 1, 1), (3, 7, 5), (130, 33, 9), (257, 5, 70), (40, 300, 3)]:
        X = rng.standard_normal((n, d))
        U = rng.standard_normal((m, d))
        pm = df.project_parallel(df.Dataset(X), U)
        assert pm.m == m and pm.n == n
        assert np.array_equal(pm.scores, orc.project(X, U))
        assert np.array_equal(df.project_naive(df.Dataset(X), U).scores, pm.scores)
    # linearity (test_projection.py:71-80), project_point cases (:82-106)
    U = rng.standard_normal((6, 4))
    a = df.project_parallel(data, U).scores
    b = df.project_parallel(df.Dataset(2.0 * x), U).scores
    assert np.array_equal(b, 2.0 * a)
    assert np.array_equal(df.project_point(np.zeros(4), U), np.zeros(6))
    z = rng.standard_normal(4)
    u = z / np.linalg.norm(z)
    assert df.project_point(z, u[None, :])[0] == pytest.approx(np.linalg.norm(z), rel=1e-14)
    assert np.array_equal(df.project_point(x[2], U), df.project_naive(df.Dataset(x[2]), U).scores[:, 0])
    with pytest.raises(df.DimensionMismatch):
        df.project_point(np.zeros(3), U)
    with pytest.raises(ValueError):
        df.Dataset(np.array([[0.0, np.nan]]))
    with pytest.raises(ValueError):
        df.Dataset(np.empty((0, 3)))
    assert df.Dataset(np.arange(3.0)).x.shape == (1, 3)


# -------------------------------------------- test_philox_directions.py cases --
def test_substreams(depthforge, orc):
    df = depthforge
    s = df.SubStream(seed=123456789123, refinement=7, query=4_000_000_001, index=5)
    u = s.uniforms(300, offset=11)
    assert np.all((u > 0.0) & (u < 1.0))
    assert np.array_equal(u, s.uniforms(300, offset=11))
    want = orc.uniforms(123456789123, np.arange(11, 311), np.full(300, 5), 7, 4_000_000_001)
    assert np.array_equal(u, want)
    g = s.normals(300, offset=11)
    assert np.array_equal(g, orc.ndtri(want))
    other = df.SubStream(seed=123456789123, refinement=7, query=4_000_000_001, index=6).uniforms(300, offset=11)
    assert not np.any(other == u)


def test_random_sphere(depthforge):
    df = depthforge
    for i in range(5):
        v = df.random_sphere(1, df.SubStream(seed=i))
        assert v.shape == (1,) and abs(v[0]) == 1.0
    rows = np.stack([df.random_sphere(7, df.SubStream(seed=3, index=i)) for i in range(200)])
    assert np.allclose(np.linalg.norm(rows, axis=1), 1.0, atol=1e-14)
    assert np.abs(rows.mean(axis=0)).max() < 0.25  # coordinate means near 0
    with pytest.raises(ValueError):
        df.random_sphere(0, df.SubStream(seed=1))


def test_caps_and_pole_streams(depthforge):
    df = depthforge
    with pytest.raises(ValueError):
        df.Pole(np.array([1.0, 1.0]))
    rng = np.random.default_rng(9)
    p = rng.standard_normal(6)
    p /= np.linalg.norm(p)
    cap = df.CapSpec(df.Pole(p), 0.4)
    batch = df.generate_batch(cap, 50, seed=17, refinement=3, query=2).directions
    assert np.allclose(np.linalg.norm(batch, axis=1), 1.0, atol=1e-14)
    assert np.all(np.arccos(np.clip(batch @ p, -1, 1)) <= 0.4 + 1e-12)  # cap membership
    # rows match scalar substreams (test_philox_directions.py:167-175)
    for j in (0, 1, 31, 49):
        row = df.random_sphere_pole(cap, df.SubStream(seed=17, refinement=3, query=2, index=j))
        assert np.array_equal(row, batch[j])
    # prefix stability under m (:177-181)
    assert np.array_equal(df.generate_batch(cap, 20, seed=17, refinement=3, query=2).directions, batch[:20])
    with pytest.raises(ValueError):
        df.generate_batch(cap, 0, seed=1, refinement=0)
    # d = 1 returns the pole; antipodal pole negates u1 (:138-146)
    one = df.generate_batch(df.CapSpec(df.Pole(np.array([-1.0])), 0.3), 4, seed=1, refinement=0).directions
    assert np.array_equal(one, np.full((4, 1), -1.0))
    e1 = np.zeros(3)
    e1[0] = 1.0
    a = df.generate_batch(df.CapSpec(df.Pole(e1), 0.7), 16, seed=5, refinement=1).directions
    b = df.generate_batch(df.CapSpec(df.Pole(-e1), 0.7), 16, seed=5, refinement=1).directions
    assert np.array_equal(b[:, 0], -a[:, 0]) and np.array_equal(b[:, 1:], a[:, 1:])
    # identity pole keeps the polar angle: u[0] == cos(theta) (:110-118)
    s = df.SubStream(seed=5, refinement=1, index=0)
    # (device cos vs glibc cos: <= 1 ulp)
    assert a[0, 0] == pytest.approx(math.cos(s.uniforms(1)[0] * 0.7), rel=3e-16, abs=0.0)


# ------------------------------------------------ test_optimizer.py cases --
def test_optimizer_cases(depthforge):
    df = depthforge
    rng = np.random.default_rng(2)
    X = rng.standard_normal((120, 3))
    data = df.Dataset(X)
    cfg = df.RrsConfig(total_directions=600, refinements=6, shrink=0.8, notion="halfspace", seed=4)
    one = df.Dataset(np.array([[1.0, 2.0, 3.0]]))
    assert df.refined_random_search(np.array([1.0, 2.0, 3.0]), one, cfg).depth == 1.0
    assert df.refined_random_search(np.full(3, 100.0), data, cfg).depth == 0.0
    res = df.refined_random_search(X[0] * 0.1, data, cfg)
    best = [t.best_depth for t in res.trace]
    assert all(a >= b for a, b in zip(best, best[1:]))
    assert [t.epsilon for t in res.trace] == [math.pi / 2 * 0.8 ** l for l in range(6)]
    assert res.directions_used == 600 and abs(np.linalg.norm(res.argmin_direction) - 1) < 1e-12
    # simple random search = one refinement (:78-88)
    srs = df.simple_random_search(X[1] * 0.5, data, k=300, notion="projection", seed=9)
    rrs = df.refined_random_search(X[1] * 0.5, data, df.RrsConfig(total_directions=300, refinements=1,
                                                                   shrink=0.5, notion="projection", seed=9))
    assert srs.depth == rrs.depth
    with pytest.raises(df.DimensionMismatch):
        df.refined_random_search(np.zeros(2), data, cfg)
    for bad in (dict(total_directions=3, refinements=4), dict(refinements=0), dict(shrink=1.0),
                dict(notion="tukey"), dict(pole_update="sometimes")):
        with pytest.raises(ValueError):
            df.RrsConfig(**bad)
    # repeat, batch-of-one, batch = sequential with query_index, permutation (:137-192)
    Z = np.concatenate([X[:5], 0.3 * X[5:9]])
    base = df.depth_batch(list(Z), data, cfg)
    again = df.depth_batch(list(Z), data, cfg)
    assert [r.depth for r in base] == [r.depth for r in again]
    for i in (0, 4, 8):
        single = df.refined_random_search(Z[i], data, cfg, query_index=i)
        assert single.depth == base[i].depth
        assert np.array_equal(single.argmin_direction, base[i].argmin_direction)
    assert df.depth_batch([Z[0]], data, cfg)[0].depth == base[0].depth
    with pytest.raises(df.DimensionMismatch, match="query 1 has dimension 2"):
        df.depth_batch([Z[0], np.zeros(2)], data, cfg)
    # pole update rule (:201-215)
    u, w = np.array([1.0, 0.0]), np.array([0.0, 1.0])
    assert df.pole_update_rule((0.3, u), (0.4, w))[1] is u
    assert df.pole_update_rule((0.3, u), (0.3, w))[1] is u
    assert df.pole_update_rule((0.3, u), (0.2, w))[1] is w
    # per_direction mode reaches the same minimum (:217-229)
    cfg2 = df.RrsConfig(total_directions=600, refinements=6, shrink=0.8, notion="halfspace", seed=4,
                        pole_update="per_direction")
    assert [r.depth for r in df.depth_batch(list(Z), data, cfg2)] == [r.depth for r in base]


def test_2d_halfspace_bounds_exact_depth(depthforge):
    """test_optimizer.py:231-251 / test_acceptance.py:194-220: in 2-D, RRS
    with k = 1e4, r = 20 is within [exact, exact + 1/n] for >= 95% of cases."""
    df = depthforge
    rng = np.random.default_rng(12)
    ok = 0
    cases = 40
    for c in range(cases):
        X = rng.standard_normal((200, 2))
        z = rng.standard_normal(2) * 0.7
        # exact 2-D halfspace depth: min over the angular sweep of closed halfplanes
        a = np.arctan2(X[:, 1] - z[1], X[:, 0] - z[0])
        cand = np.concatenate([a + np.pi / 2, a - np.pi / 2])
        best = 200
        for t in cand:
            for eps in (1e-9, -1e-9):
                u = np.array([np.cos(t + eps), np.sin(t + eps)])
                best = min(best, int(np.count_nonzero((X - z) @ u >= 0)))
        exact = best / 200
        cfg = df.RrsConfig(total_directions=10_000, refinements=20, shrink=0.9, notion="halfspace", seed=c)
        got = df.refined_random_search(z, df.Dataset(X), cfg).depth
        ok += exact <= got + 1e-12 and got <= exact + 1 / 200 + 1e-12
    assert ok >= 0.95 * cases
