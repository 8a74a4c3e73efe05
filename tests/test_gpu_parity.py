"""Parity of the CUDA path (through the C ABI) against the reference fixtures
and the CPU oracle.  Three tiers (BASELINE.json north_star):

  1. halfspace counts bit-exact except inside the tie zone
     |<u,x_i> - <u,z>| < 1e-6 * max(|x_i|, |z|), whose size is logged;
  2. per-direction projection / asymmetric-projection depths within 1e-5 rel;
  3. end-to-end RRS depths: Kendall tau >= 0.99 at equal hyperparameters
     (plus exact count equality on the config-4 shape).
"""

import numpy as np
import pytest
from scipy.stats import kendalltau

pytestmark = pytest.mark.gpu

TIE_REL = 1e-6
DEPTH_RTOL = 1e-5


PATHS = ["ffma", "tensor", "filter"]


class contract_path:
    """Force the halfspace contraction kernel (FFMA or tcgen05) for a block."""

    def __init__(self, pkg, path):
        self.eng, self.path = pkg.engine(), path

    def __enter__(self):
        self.eng.set_contract_path(self.path)

    def __exit__(self, *exc):
        self.eng.set_contract_path("auto")


def tie_zone(X, z, U):
    px = X @ U.T  # (n, m) FP64
    pz = U @ z
    scale = np.maximum(np.linalg.norm(X, axis=1)[:, None], np.linalg.norm(z))
    return (np.abs(px - pz[None, :]) < TIE_REL * scale).sum(axis=0)


def test_philox_kats_on_device(b200):
    eng = b200.engine()
    z = eng.philox4x32(np.zeros((4, 1), dtype=np.uint32), 0, 0)[:, 0]
    assert [int(w) for w in z] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    ones = eng.philox4x32(np.full((4, 1), 0xFFFFFFFF, dtype=np.uint32), 0xFFFFFFFF, 0xFFFFFFFF)[:, 0]
    assert [int(w) for w in ones] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    ctr = np.array([[0x243F6A88], [0x85A308D3], [0x13198A2E], [0x03707344]], dtype=np.uint32)
    pi = eng.philox4x32(ctr, 0xA4093822, 0x299F31D0)[:, 0]
    assert [int(w) for w in pi] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_philox_words_bitexact(b200, golden):
    k0, k1 = (int(k) for k in golden["philox_key"])
    got = b200.engine().philox4x32(golden["philox_ctr"], k0, k1)
    assert np.array_equal(got, golden["philox_out"])


def test_cap_directions_match_reference(b200, golden):
    """Device generate_batch rows vs the reference rows (FP64; CUDA cos/log
    may differ from glibc by an ulp)."""
    eng = b200.engine()
    worst = 0.0
    for i in range(int(golden["cap_count"])):
        p = golden[f"cap{i}_pole"]
        eps, m, seed, l, q = golden[f"cap{i}_args"]
        U = eng.cap_directions(p, eps, int(m), int(seed), int(l), int(q))
        ref = golden[f"cap{i}_U"]
        worst = max(worst, float(np.max(np.abs(U - ref))))
        assert np.all(np.abs(np.linalg.norm(U, axis=1) - 1.0) <= 1e-12)
        assert np.all(U @ p >= np.cos(eps) - 1e-10)  # cap membership
    print(f"max |U_gpu - U_ref| = {worst:.3e}")
    assert worst <= 1e-13


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("tag", ["ed_small", "ed_cauchy"])
def test_tier1_halfspace_counts(b200, golden, tag, path):
    X, U, Z = golden[f"{tag}_x"], golden[f"{tag}_U"], golden[f"{tag}_Z"]
    data = b200.Dataset(X)
    total_zone = used = 0
    for qi, z in enumerate(Z):
        with contract_path(b200, path):
            out, cle, cge = b200.evaluate_directions_counts(z, data, U)
        rcle, rcge = golden[f"{tag}_cle"][qi], golden[f"{tag}_cge"][qi]
        T = tie_zone(X, z, U)
        total_zone += int(T.sum())
        dle, dge = np.abs(cle - rcle), np.abs(cge - rcge)
        assert np.all(dle <= T) and np.all(dge <= T), (qi, np.flatnonzero((dle > T) | (dge > T)))
        used += int(np.count_nonzero((dle > 0) | (dge > 0)))
        ref_depth = golden[f"{tag}_halfspace"][qi]
        exact = (dle == 0) & (dge == 0)
        assert np.array_equal(out[exact], ref_depth[exact])
    print(f"{tag}/{path}: tie-zone elements {total_zone}, directions using slack {used}")


@pytest.mark.parametrize("path", PATHS)
def test_self_tie_in_sample(b200, golden, path):
    """z = x_i: the query's own row projects to exactly 0 (difference form), so
    it is counted on both sides of every direction."""
    X, U = golden["ed_small_x"], golden["ed_small_U"]
    data = b200.Dataset(X)
    for i in (0, 7, 123):
        with contract_path(b200, path):
            _, cle, cge = b200.evaluate_directions_counts(X[i], data, U)
        assert np.all(cle >= 1) and np.all(cge >= 1)
        assert np.all(cle + cge >= X.shape[0] + 1)


@pytest.mark.parametrize("tag", ["ed_small", "ed_cauchy"])
@pytest.mark.parametrize("notion", ["projection", "asym_projection"])
def test_tier2_projection_depths(b200, golden, tag, notion):
    X, U, Z = golden[f"{tag}_x"], golden[f"{tag}_U"], golden[f"{tag}_Z"]
    data = b200.Dataset(X)
    cfg = b200.ParallelConfig(workers=1)
    for qi, z in enumerate(Z):
        got = b200.evaluate_directions(z, data, U, notion, cfg)
        np.testing.assert_allclose(got, golden[f"{tag}_{notion}"][qi], rtol=DEPTH_RTOL, atol=0)


@pytest.mark.parametrize("n", [1, 2, 3, 18, 101, 1024])
def test_univariate_spans_tie_heavy(b200, golden, n):
    """The reference's tie-heavy span cases (test_backends.py:59-73) through the
    fused device path: d = 1, u = 1, so y = x - z."""
    px, pz = golden[f"span_n{n}_px"], golden[f"span_n{n}_pz"]
    U = np.ones((1, 1))
    cfg = b200.ParallelConfig(workers=1)
    for name in ("halfspace", "projection", "asym_projection"):
        ref = golden[f"span_n{n}_{name}"]
        got = np.array([b200.evaluate_directions(pz[j:j + 1], b200.Dataset(px[j][:, None]), U, name, cfg)[0]
                        for j in range(px.shape[0])])
        if name == "halfspace":
            assert np.array_equal(got, ref)
        else:
            np.testing.assert_allclose(got, ref, rtol=DEPTH_RTOL, atol=0)


def test_degenerate_rows(b200, golden):
    px, pz = golden["degen_px"], golden["degen_pz"]
    cfg = b200.ParallelConfig(workers=1)
    for name in ("halfspace", "projection", "asym_projection"):
        got = [b200.evaluate_directions(pz[j:j + 1], b200.Dataset(px[j][:, None]), np.ones((1, 1)), name,
                                        cfg)[0] for j in range(3)]
        assert np.array_equal(np.array(got), golden[f"degen_{name}"]), name


@pytest.mark.parametrize("path", PATHS)
def test_tier3_config1_all_points(b200, golden, path):
    """BASELINE config 1: halfspace, n=1000, d=5, k=1000, r=10, alpha=0.9, seed 1."""
    X = golden["c1_x"]
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=1000, refinements=10, shrink=0.9, notion="halfspace", seed=1)
    with contract_path(b200, path):
        depth, argmin, tr, cnt = b200.depth_batch_arrays(X, data, cfg, trace=True)
    ref = golden["c1_depth"]
    same = np.mean(depth == ref)
    tau = kendalltau(depth, ref).statistic
    print(f"config 1 ({path}): {same:.4f} of depths identical, tau = {tau:.5f}")
    assert tau >= 0.99
    assert same >= 0.98
    assert np.array_equal(np.rint(depth * X.shape[0]).astype(np.int64), cnt)
    assert np.all(np.abs(np.linalg.norm(argmin, axis=1) - 1.0) <= 1e-12)
    eps = np.array(cfg.epsilons())
    assert np.array_equal(tr[:, :, 1], np.broadcast_to(eps, tr[:, :, 1].shape))  # exact schedule
    assert np.all(np.diff(tr[:, :, 0], axis=1) <= 0)  # monotone trace


@pytest.mark.parametrize("notion", ["halfspace", "projection", "asym_projection"])
def test_tier3_small_rrs(b200, golden, notion):
    X, Z = golden[f"rrs_{notion}_x"], golden[f"rrs_{notion}_z"]
    cfg = b200.RrsConfig(total_directions=400, refinements=8, shrink=0.8, notion=notion, seed=77)
    res = b200.depth_batch(list(Z), b200.Dataset(X), cfg)
    depth = np.array([r.depth for r in res])
    ref = golden[f"rrs_{notion}_depth"]
    if notion == "halfspace":
        assert np.mean(depth == ref) >= 0.9
    else:
        close = np.isclose(depth, ref, rtol=DEPTH_RTOL, atol=0)
        assert np.mean(close) >= 0.9
    assert kendalltau(depth, ref).statistic >= 0.99
    for r in res:
        assert len(r.trace) == 8 and r.directions_used == 400
        assert all(t.epsilon == (np.pi / 2) * 0.8**l for l, t in enumerate(r.trace))


@pytest.mark.parametrize("path", PATHS)
def test_config4_miniature_exact_counts(b200, golden, path):
    X, Z = golden["c4mini_x"], golden["c4mini_z"]
    cfg = b200.RrsConfig(total_directions=2000, refinements=20, shrink=0.9, notion="halfspace", seed=1)
    with contract_path(b200, path):
        depth, _, _, cnt = b200.depth_batch_arrays(Z, b200.Dataset(X), cfg)
    ref = golden["c4mini_depth"]
    n = X.shape[0]
    assert np.array_equal(cnt[:6], np.ones(6, dtype=np.int64))  # in-sample: self-tie only
    assert np.array_equal(depth[:6], ref[:6])
    rc = np.rint(ref * n).astype(np.int64)
    assert np.all(np.abs(cnt - rc) <= np.maximum(1, rc // 50)), (cnt, rc)


def test_shard_offsets_bitwise(b200, golden):
    """Global query indices make results independent of how queries are split."""
    X = golden["c1_x"]
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=1000, refinements=10, shrink=0.9, notion="halfspace", seed=1)
    full = b200.depth_batch_arrays(X[:96], data, cfg)
    parts = [b200.depth_batch_arrays(X[a:a + 24], data, cfg, q0=a) for a in range(0, 96, 24)]
    assert np.array_equal(full[0], np.concatenate([p[0] for p in parts]))
    assert np.array_equal(full[1], np.concatenate([p[1] for p in parts]))


def test_structure_cases(b200):
    data = b200.Dataset([[0.3, -0.7]])
    assert b200.simple_random_search(data.x[0], data, 50, "halfspace", 0).depth == 1.0
    rng = np.random.default_rng(1)
    data = b200.Dataset(rng.standard_normal((100, 3)))
    assert b200.simple_random_search(np.full(3, 1e6), data, 32, "halfspace", 1).depth == 0.0


def test_datadepth_wrappers(b200, golden):
    X = golden["rrs_halfspace_x"]
    Z = golden["rrs_halfspace_z"]
    for fn, notion in ((b200.halfspace, "halfspace"), (b200.projection, "projection"),
                       (b200.aprojection, "asym_projection")):
        got = fn(Z, X, NRandom=400, n_refinements=8, sphcap_shrink=0.8, solver="refinedrandom", seed=77)
        cfg = b200.RrsConfig(total_directions=400, refinements=8, shrink=0.8, notion=notion, seed=77)
        ref = b200.depth_batch_arrays(Z, b200.Dataset(X), cfg)[0]
        assert np.array_equal(got, ref)
    with pytest.raises(ValueError):
        b200.halfspace(Z, X, solver="neldermead")


@pytest.mark.parametrize("path", PATHS)
def test_paths_agree_on_counts(b200, path):
    """Both contraction kernels against the FP64 oracle on random data with
    off-sample queries (n not a multiple of the 128-point tile, m not a
    multiple of the direction blocks)."""
    from oracle import oracle

    rng = np.random.default_rng(21)
    X = rng.standard_normal((5000 + 77, 37))
    U = rng.standard_normal((300, 37))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    slack = 0
    for z in (X[5], 0.2 * X[9], rng.standard_normal(37)):
        with contract_path(b200, path):
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        _, rle, rge = oracle.evaluate_directions(z, X, U, "halfspace", with_counts=True)
        T = tie_zone(X, z, U)
        assert np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T)
        slack += int(np.count_nonzero((cle != rle) | (cge != rge)))
    print(f"{path}: directions using tie-zone slack {slack} / 900")


@pytest.mark.slow
def test_config4_scale_in_sample_counts(b200):
    """Config 4 at full size (n=100k, d=50, k=20000, r=20) on a few in-sample
    queries: every depth is exactly 1/n (self-tie only)."""
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    X = toeplitz_gaussian(50, 100_000, seed=0)
    cfg = b200.RrsConfig(total_directions=20_000, refinements=20, shrink=0.9, notion="halfspace", seed=1)
    idx = np.array([0, 12345, 99_999])
    depth, _, _, cnt = b200.depth_batch_arrays(X[idx], b200.Dataset(X), cfg, q0=0)
    assert np.array_equal(cnt, np.ones(3, dtype=np.int64))
    assert np.all(depth == 1.0 / 100_000)


@pytest.mark.parametrize("dist", ["gaussian", "cauchy"])
def test_tier1_config4_scale_counts(b200, orc, dist):
    """Tier 1 at the config-4 shape (n=100k, d=50, 1000 directions): counts
    from every contraction kernel equal the reference's counts except inside
    the tie zone, for in-sample, off-sample and near-duplicate queries.  The
    checker is the pinned oracle (the reference's FP64 no-FMA projections
    and ``_kernels.pyx`` counting, self-tie exact), so "directions using
    slack" measures GPU error only."""
    from paper_2506_08262_b200.synthetic import student_t, toeplitz_gaussian

    X = toeplitz_gaussian(50, 100_000, seed=0) if dist == "gaussian" else student_t(50, 100_000, 1.0, seed=0)
    rng = np.random.default_rng(8)
    U = rng.standard_normal((1000, 50))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    xn = np.linalg.norm(X, axis=1)
    px = orc.project(X, U)  # (m, n), the reference's arithmetic
    slack = {p: 0 for p in PATHS}
    zone_total = 0
    for z in (X[3], 0.3 * X[7], np.zeros(50), X[11] + 1e-3 * rng.standard_normal(50)):
        _, rle, rge = orc.univariate("halfspace", px, orc.project_point(z, U), with_counts=True)
        y = px - orc.project_point(z, U)[:, None]
        T = (np.abs(y) < TIE_REL * np.maximum(xn[None, :], np.linalg.norm(z))).sum(axis=1)
        zone_total += int(T.sum())
        for path in PATHS:
            with contract_path(b200, path):
                _, cle, cge = b200.evaluate_directions_counts(z, data, U)
            bad = np.flatnonzero((np.abs(cle - rle) > T) | (np.abs(cge - rge) > T))
            assert bad.size == 0, (path, bad)
            slack[path] += int(np.count_nonzero((cle != rle) | (cge != rge)))
    print(f"config-4 shape {dist}: tie-zone elements {zone_total}, directions using slack "
          f"{slack} / 4000")


@pytest.mark.parametrize("d", [1, 3, 16, 22, 27, 44, 50, 59, 61, 64])
def test_tensor_layout_dims(b200, d):
    """The packed split-product K layout (kernels.h tc_layout) for every shape of
    remainder: d % 16 = 0 (no tail step), 3 (one), 6 (two), 11/12 (three tail
    steps), d < 16 (tail only) -- tensor-path counts against FP64 within the
    tie zone, n not a multiple of the 128-point tile, m not a multiple of 128."""
    rng = np.random.default_rng(100 + d)
    X = rng.standard_normal((4096 + 203, d)) * rng.uniform(0.1, 10.0, size=d)
    U = rng.standard_normal((333, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    xn = np.linalg.norm(X, axis=1)
    for z in (X[17], 0.5 * X[3] + 0.5 * X[4], np.full(d, 0.1)):
        with contract_path(b200, "tensor"):
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        y = X @ U.T - (U @ z)[None, :]
        T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
        rle, rge = (y <= 0).sum(axis=0), (y >= 0).sum(axis=0)
        assert np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T), d


@pytest.mark.parametrize("d", [65, 72, 100, 123, 128, 129, 150, 187, 200, 253, 256])
def test_tensor_wide_dims(b200, d):
    """The wide tensor path (64 < d <= 256: the pre-split contract_tcp.cu by
    default, 64-coordinate slices, one or two accumulator buffers; d = 123 /
    187 / 253: a last slice of 59..63 coordinates, 9 stored K steps and as many
    MMAs as a full slice; d = 253: one accumulator) against FP64
    within the tie zone and against the FFMA kernel, with a near-duplicate
    query, an in-sample query (self tie) and heterogeneous coordinate scales;
    n not a multiple of the tile, m not of the block."""
    rng = np.random.default_rng(300 + d)
    X = rng.standard_normal((4096 + 77, d)) * rng.uniform(0.1, 10.0, size=d)
    U = rng.standard_normal((200, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    xn = np.linalg.norm(X, axis=1)
    for z in (X[5], X[9] + 1e-4 * rng.standard_normal(d), np.full(d, 0.2)):
        with contract_path(b200, "tensor"):
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        with contract_path(b200, "ffma"):
            _, fle, fge = b200.evaluate_directions_counts(z, data, U)
        y = X @ U.T - (U @ z)[None, :]
        T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
        rle, rge = (y <= 0).sum(axis=0), (y >= 0).sum(axis=0)
        assert np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T), d
        assert np.all(np.abs(cle - fle) <= T) and np.all(np.abs(cge - fge) <= T), d


def test_tensor_dims_sweep(b200):
    """Every tensor-path K layout shape in one sweep: d = 1 .. 256 (every
    remainder of the last 64-coordinate slice, 1 to 4 slices, one and two
    accumulators), halfspace counts of the tensor path (contract_tc /
    contract_tcp) and the converter path (contract_tcw) against FP64 within
    the tie zone, an in-sample and an off-sample query."""
    rng = np.random.default_rng(77)
    Xall = rng.standard_normal((4096 + 45, 256))
    Uall = rng.standard_normal((72, 256))
    bad = []
    dims = sorted(set(list(range(1, 257, 5)) + [59, 61, 63, 64, 65, 123, 127, 128, 187, 191, 192, 251, 255, 256]))
    for d in dims:
        X = np.ascontiguousarray(Xall[:, :d])
        U = Uall[:, :d] / np.linalg.norm(Uall[:, :d], axis=1)[:, None]
        data = b200.Dataset(X)
        xn = np.linalg.norm(X, axis=1)
        for z in (X[11], 0.5 * X[2] + 0.3):
            y = X @ U.T - (U @ z)[None, :]
            T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
            rle, rge = (y <= 0).sum(axis=0), (y >= 0).sum(axis=0)
            for path in (("tensor", "convert") if d > 64 else ("tensor",)):
                with contract_path(b200, path):
                    _, cle, cge = b200.evaluate_directions_counts(z, data, U)
                if not (np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T)):
                    bad.append((d, path))
    assert not bad, bad


def test_tensor_tile_padding_sweep(b200):
    """Point counts around the 128-point tile and the 4096-point auto switch
    (padding rows excluded from every count, the last tile partly filled):
    tensor-path halfspace counts within the tie zone of FP64 at d = 50
    (contract_tc) and d = 120 (contract_tcp, contract_tcw), in- and
    off-sample queries."""
    rng = np.random.default_rng(80)
    Xall = rng.standard_normal((4400, 120))
    Uall = rng.standard_normal((40, 120))
    bad = []
    for n in (4096, 4097, 4223, 4224, 4225, 4351, 4352):
        for d in (50, 120):
            X = np.ascontiguousarray(Xall[:n, :d])
            U = Uall[:, :d] / np.linalg.norm(Uall[:, :d], axis=1)[:, None]
            data = b200.Dataset(X)
            xn = np.linalg.norm(X, axis=1)
            for z in (X[n - 1], 0.3 * X[0] - 0.2):
                y = X @ U.T - (U @ z)[None, :]
                T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
                for path in ("tensor", "convert") if d > 64 else ("tensor",):
                    with contract_path(b200, path):
                        _, cle, cge = b200.evaluate_directions_counts(z, data, U)
                    if not (np.all(np.abs(cle - (y <= 0).sum(axis=0)) <= T)
                            and np.all(np.abs(cge - (y >= 0).sum(axis=0)) <= T)):
                        bad.append((n, d, path))
    assert not bad, bad


def test_projection_rowlength_sweep(b200):
    """D_P / D_AP across the row lengths where the kernels switch (the FP64
    store below n = 4096, the tensor store above; select v2 below 2048, v3 with
    256 / 512 threads, v5 past 53248), auto paths, against the FP64 oracle to
    1e-5 relative."""
    from oracle import oracle

    rng = np.random.default_rng(81)
    Xall = rng.standard_normal((60_001, 20))
    U = rng.standard_normal((12, 20))
    U /= np.linalg.norm(U, axis=1)[:, None]
    bad = []
    for n in (2047, 2048, 4095, 4096, 16384, 16385, 53248, 53249, 60_001):
        X = np.ascontiguousarray(Xall[:n])
        data = b200.Dataset(X)
        z = 0.2 * X[1] + 0.05
        for notion in ("projection", "asym_projection"):
            got = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig(workers=1))
            ref = oracle.evaluate_directions(z, X, U, notion)
            if not np.allclose(got, ref, rtol=DEPTH_RTOL, atol=0):
                bad.append((n, notion))
    assert not bad, bad


def test_ffma_dims_sweep(b200):
    """The FP32 FFMA kernels over d = 1 .. 256 (contract.cu: the halfspace
    count below n = 4096 and the forced FFMA projection store): counts within
    the tie zone of FP64 and D_P depths against the oracle to 1e-5."""
    from oracle import oracle

    rng = np.random.default_rng(79)
    Xall = rng.standard_normal((3000, 256))
    Uall = rng.standard_normal((40, 256))
    bad = []
    for d in sorted(set(list(range(1, 257, 7)) + [63, 64, 65, 128, 129, 255, 256])):
        X = np.ascontiguousarray(Xall[:, :d])
        U = Uall[:, :d] / np.linalg.norm(Uall[:, :d], axis=1)[:, None]
        data = b200.Dataset(X)
        z = 0.5 * X[9] + 0.05
        y = X @ U.T - (U @ z)[None, :]
        T = (np.abs(y) < TIE_REL * np.maximum(np.linalg.norm(X, axis=1), np.linalg.norm(z))[:, None]).sum(axis=0)
        with contract_path(b200, "ffma"):
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
            got = b200.evaluate_directions(z, data, U, "projection", b200.ParallelConfig(workers=1))
        if not (np.all(np.abs(cle - (y <= 0).sum(axis=0)) <= T) and np.all(np.abs(cge - (y >= 0).sum(axis=0)) <= T)):
            bad.append((d, "counts"))
        if not np.allclose(got, oracle.evaluate_directions(z, X, U, "projection"), rtol=DEPTH_RTOL, atol=0):
            bad.append((d, "projection"))
    assert not bad, bad


def test_tensor_store_dims_sweep(b200):
    """The tensor projection stores over every K layout shape (contract_tc
    STORE for d <= 64, contract_tcp STORE above, and the three-term
    contract_tcs for d <= 50; d = 2 .. 256 in steps of 9 plus the 9-step last
    slices): D_P / D_AP per direction against the FP64 oracle to 1e-5
    relative."""
    from oracle import oracle

    rng = np.random.default_rng(78)
    Xall = rng.standard_normal((4096 + 61, 256))
    Uall = rng.standard_normal((24, 256))
    bad = []
    dims = sorted(set(list(range(2, 257, 9)) + [59, 61, 63, 123, 187, 251, 255]))
    for d in dims:
        X = np.ascontiguousarray(Xall[:, :d])
        U = Uall[:, :d] / np.linalg.norm(Uall[:, :d], axis=1)[:, None]
        data = b200.Dataset(X)
        z = 0.4 * X[5] + 0.1
        for notion in ("projection", "asym_projection"):
            ref = oracle.evaluate_directions(z, X, U, notion)
            for path in (("tensor", "tensor3") if d <= 50 else ("tensor",)):
                with contract_path(b200, path):
                    got = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig(workers=1))
                if not np.allclose(got, ref, rtol=DEPTH_RTOL, atol=0):
                    bad.append((d, notion, path, float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))))
    assert not bad, bad


@pytest.mark.parametrize("d", [50, 120])
def test_halfspace_query_batches_bitwise(b200, d):
    """A workspace that holds only a few queries splits a depth_batch into
    several engine batches (per batch: the coinciding-row lists, the state,
    the refinements): depths, argmins and counts bitwise equal to one batch,
    with and without the early exit (tensor paths: contract_tc / the pre-split
    contract_tcp)."""
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    X = toeplitz_gaussian(d, 6000, seed=4)
    Z = np.vstack([X[:20], 0.5 * X[20:37]])
    data = b200.Dataset(X)
    eng = b200.engine()
    for early in (False, True):
        cfg = b200.RrsConfig(total_directions=1200, refinements=4, shrink=0.8, notion="halfspace", seed=2,
                             early_exit=early)
        one = b200.depth_batch_arrays(Z, data, cfg)
        eng.set_workspace_limit(4 << 20)
        try:
            many = b200.depth_batch_arrays(Z, data, cfg)
        finally:
            eng.set_workspace_limit(8 << 30)
        for a_, b_ in zip(one, many):
            assert np.array_equal(a_, b_)


@pytest.mark.parametrize("d", [80, 200, 253])
def test_presplit_vs_converter(b200, d):
    """The pre-split wide kernel (contract_tcp.cu: query applied in the epilogue
    as y = acc inv_i + <u, -z>, coinciding rows excluded by index) against FP64
    and against the converter kernel (contract_path 'convert', contract_tcw.cu)
    on the cases the index exclusion and the epilogue shift must get right:
    a query with 3 duplicated rows, one with more duplicates than the list
    holds (TCP_COIN_MAX = 64: the batch goes to the converter kernel), a far
    query, an all-zero query against data containing zero rows, and data far
    from the origin."""
    rng = np.random.default_rng(500 + d)
    n = 5000 + 33
    base = rng.standard_normal((n, d))
    cases = []
    X = base.copy()
    X[10:13] = X[7]  # X[7] occurs 4 times
    cases.append((X, X[7]))
    X = base.copy()
    X[100:170] = X[99]  # 71 copies: past the coinciding-row list
    cases.append((X, X[99]))
    cases.append((base, base[3] + 1e3))
    X = base.copy()
    X[20:25] = 0.0
    cases.append((X, np.zeros(d)))
    X = base + 500.0
    cases.append((X, X[11]))
    U = rng.standard_normal((300, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    for X, z in cases:
        data = b200.Dataset(X)
        with contract_path(b200, "tensor"):
            _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        with contract_path(b200, "convert"):
            _, vle, vge = b200.evaluate_directions_counts(z, data, U)
        y = X @ U.T - (U @ z)[None, :]
        xn = np.linalg.norm(X, axis=1)
        T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
        exact = np.all(X == z[None, :], axis=1).sum()  # rows coinciding with z: ties on both sides
        rle, rge = (y <= 0).sum(axis=0), (y >= 0).sum(axis=0)
        assert np.all(cle >= exact) and np.all(cge >= exact)
        assert np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T)
        assert np.all(np.abs(cle - vle) <= T) and np.all(np.abs(cge - vge) <= T)


def test_tensor_wide_rrs_matches_ffma(b200):
    """Full RRS at d = 200 (wide tensor path) against the FFMA path: identical
    depths unless a count sits in the tie zone (Kendall tau over queries)."""
    rng = np.random.default_rng(11)
    X = rng.standard_normal((6000, 200))
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=600, refinements=3, shrink=0.9, notion="halfspace", seed=4)
    with contract_path(b200, "tensor"):
        dt = b200.depth_batch_arrays(X[:24], data, cfg)[0]
    with contract_path(b200, "ffma"):
        df = b200.depth_batch_arrays(X[:24], data, cfg)[0]
    with contract_path(b200, "convert"):
        dc = b200.depth_batch_arrays(X[:24], data, cfg)[0]
    assert np.mean(dt == df) >= 0.9 and kendalltau(dt, df)[0] >= 0.95
    assert np.mean(dt == dc) >= 0.9 and kendalltau(dt, dc)[0] >= 0.95


@pytest.mark.parametrize("notion", ["projection", "asym_projection"])
@pytest.mark.parametrize("n", [53248, 60000, 60001])
def test_tier2_large_rows(b200, notion, n):
    """Rows at the shared-memory limit of the select kernel and past it (the
    global-memory select paths: keys streamed in place for n % 4 == 0, the
    11-bit legacy kernel otherwise), Cauchy data, against the FP64 oracle."""
    from oracle import oracle
    from paper_2506_08262_b200.synthetic import student_t

    X = student_t(7, n, 1.0, seed=3)
    rng = np.random.default_rng(4)
    U = rng.standard_normal((16, 7))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    cfg = b200.ParallelConfig(workers=1)
    for z in (X[5], np.median(X, axis=0) + 0.1):
        got = b200.evaluate_directions(z, data, U, notion, cfg)
        ref = oracle.evaluate_directions(z, X, U, notion)
        np.testing.assert_allclose(got, ref, rtol=DEPTH_RTOL, atol=0)


@pytest.mark.parametrize("notion", ["halfspace", "projection"])
def test_config5_shape(b200, notion):
    """The config-5 shape class (d = 200: the wide tensor contraction for
    halfspace, the FFMA centred store for projection; n past the shared-memory
    select: global-memory select) at n = 400k, Cauchy data, 48 directions,
    against FP64: halfspace counts within the tie zone, projection depths to
    DEPTH_RTOL."""
    from oracle import oracle
    from paper_2506_08262_b200.synthetic import student_t

    X = student_t(200, 400_000, 1.0, seed=5)
    rng = np.random.default_rng(6)
    U = rng.standard_normal((48, 200))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    z = X[9] + 0.01 * rng.standard_normal(200)
    if notion == "halfspace":
        _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        y = X @ U.T - (U @ z)[None, :]
        xn = np.linalg.norm(X, axis=1)
        T = (np.abs(y) < TIE_REL * np.maximum(xn, np.linalg.norm(z))[:, None]).sum(axis=0)
        rle, rge = (y <= 0).sum(axis=0), (y >= 0).sum(axis=0)
        assert np.all(np.abs(cle - rle) <= T) and np.all(np.abs(cge - rge) <= T)
    else:
        got = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig(workers=1))
        ref = oracle.evaluate_directions(z, X, U, notion)
        np.testing.assert_allclose(got, ref, rtol=DEPTH_RTOL, atol=0)


def test_dataset_validation_on_device(b200):
    """The C ABI validates datasets on the device copy (host and device entry
    points): non-finite entries and |x| > 1e38 are refused with the
    reference's message, and the engine keeps its previous dataset."""
    import torch

    eng = b200.engine()
    rng = np.random.default_rng(2)
    X = rng.standard_normal((5000, 4))
    data = b200.Dataset(X)
    U = rng.standard_normal((16, 4))
    U /= np.linalg.norm(U, axis=1)[:, None]
    before = b200.evaluate_directions(X[3], data, U, "projection", b200.ParallelConfig(workers=1))
    for bad, msg in ((np.nan, "non-finite"), (np.inf, "non-finite"), (3e38, "FP32 contraction range")):
        Y = X.copy()
        Y[4321, 2] = bad
        with pytest.raises(ValueError, match=msg):
            eng.set_dataset(Y, key=object())
        with pytest.raises(ValueError, match=msg):
            eng.set_dataset_device(torch.from_numpy(Y).cuda(), key=object())
    eng.set_dataset(X, key=data._token)  # the previous dataset object is still served
    after = b200.evaluate_directions(X[3], data, U, "projection", b200.ParallelConfig(workers=1))
    np.testing.assert_array_equal(before, after)


@pytest.mark.parametrize("store", ["tensor", "tensor3"])
@pytest.mark.parametrize("notion", ["projection", "asym_projection"])
@pytest.mark.parametrize("shape", [(10_000, 20, "gaussian"), (50_000, 50, "cauchy"), (53_248, 7, "cauchy"),
                                   (4_097, 33, "gaussian"), (60_001, 48, "cauchy"), (30_000, 90, "cauchy"),
                                   (20_000, 256, "gaussian"), (12_000, 64, "cauchy"), (9_000, 253, "gaussian"),
                                   (6_000, 123, "gaussian"), (8_000, 61, "gaussian")])
def test_tensor_store_projection_depths(b200, notion, shape, store):
    """The tensor-core projection stores of the centred frame: "tensor" = the
    two-term FP16 split (contract_tc.cu STORE for d <= 64, the pre-split
    contract_tcp.cu STORE above; round 1's uncentred frame lost 1e-5 with it on
    Cauchy rows),
    "tensor3" = the three-term split (contract_tcs.cu, d <= 50): per-direction
    D_P / D_AP against the FP64 oracle to the north_star's 1e-5 relative, at the
    config-2 / config-3 shapes, odd n and d, far queries, shared-memory and
    global-memory select rows."""
    from oracle import oracle
    from paper_2506_08262_b200.synthetic import student_t, toeplitz_gaussian

    n, d, dist = shape
    X = toeplitz_gaussian(d, n, seed=1) if dist == "gaussian" else student_t(d, n, 1.0, seed=1)
    rng = np.random.default_rng(n + d)
    U = rng.standard_normal((24, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    cfg = b200.ParallelConfig(workers=1)
    if store == "tensor3" and d > 50:
        pytest.skip("the three-term split store covers d <= 50")
    for z in (X[7], np.median(X, axis=0) + 0.05, -3.0 * X[11]):
        with contract_path(b200, store):
            got = b200.evaluate_directions(z, data, U, notion, cfg)
        ref = oracle.evaluate_directions(z, X, U, notion)
        np.testing.assert_allclose(got, ref, rtol=DEPTH_RTOL, atol=0)


def test_tensor_store_rrs_matches_ffma(b200):
    """Full projection-depth RRS at the config-3 shape with the tensor store
    against the FFMA store: per-query depths within the north_star tolerance
    unless a pole update flipped on a near-tie (Kendall tau >= 0.99)."""
    from paper_2506_08262_b200.synthetic import student_t

    X = student_t(50, 20_000, 1.0, seed=0)
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=400, refinements=4, shrink=0.9, notion="asym_projection", seed=2)
    with contract_path(b200, "ffma"):
        df = b200.depth_batch_arrays(X[:32], data, cfg)[0]
    for store in ("tensor", "tensor3"):
        with contract_path(b200, store):
            dt = b200.depth_batch_arrays(X[:32], data, cfg)[0]
        close = np.isclose(dt, df, rtol=1e-5, atol=0)
        assert close.mean() >= 0.9 and kendalltau(dt, df)[0] >= 0.99, store


@pytest.mark.parametrize("path", ["ffma", "tensor", "tensor3"])
@pytest.mark.parametrize("d", [40, 120])
def test_store_direction_chunks_bitwise(b200, path, d):
    """A workspace too small for a query's projections splits the store into
    direction chunks (engine jchunk < blocks per query) and batches of one
    query: depths bitwise equal to the unchunked run, for the FFMA and the
    tensor-core stores (d = 120: the pre-split contract_tcp STORE)."""
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    if path == "tensor3" and d > 50:
        pytest.skip("the three-term split store covers d <= 50")
    X = toeplitz_gaussian(d, 10_000, seed=2)
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=2000, refinements=2, shrink=0.9, notion="projection", seed=5)
    eng = b200.engine()
    with contract_path(b200, path):
        full = b200.depth_batch_arrays(X[:6], data, cfg)
        eng.set_workspace_limit(64 << 20)  # y budget 32 MB < 1024 x 10k x 4 per query
        try:
            chunked = b200.depth_batch_arrays(X[:6], data, cfg)
        finally:
            eng.set_workspace_limit(8 << 30)
    np.testing.assert_array_equal(full[0], chunked[0])
    np.testing.assert_array_equal(full[1], chunked[1])


@pytest.mark.parametrize("n", [1, 5, 130])
@pytest.mark.parametrize("d", [20, 90, 200])
def test_tensor_paths_tiny_n(b200, n, d):
    """Tensor paths forced on tiny datasets (one partly padded tile, a single
    point): halfspace counts (contract_tc / contract_tcp) exact against FP64
    outside the tie zone, projection depths (contract_tcs for d <= 50, FFMA
    store above) against the oracle."""
    from oracle import oracle

    rng = np.random.default_rng(n * 1000 + d)
    X = rng.standard_normal((n, d))
    U = rng.standard_normal((40, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    z = X[0] + 0.1 * rng.standard_normal(d)
    with contract_path(b200, "tensor"):
        _, cle, cge = b200.evaluate_directions_counts(z, data, U)
        got = b200.evaluate_directions(z, data, U, "projection", b200.ParallelConfig(workers=1))
    y = X @ U.T - (U @ z)[None, :]
    T = (np.abs(y) < TIE_REL * np.maximum(np.linalg.norm(X, axis=1), np.linalg.norm(z))[:, None]).sum(axis=0)
    assert np.all(np.abs(cle - (y <= 0).sum(axis=0)) <= T) and np.all(np.abs(cge - (y >= 0).sum(axis=0)) <= T)
    # d > 50 at these sizes takes the FP64-accumulated centred store (center.cu):
    # the MAD of a handful of points can sit far below the projections' spread
    np.testing.assert_allclose(got, oracle.evaluate_directions(z, X, U, "projection"), rtol=DEPTH_RTOL, atol=0)


@pytest.mark.parametrize("d", [257, 384, 1024])
def test_wide_dimensions(b200, d):
    """d > 256 (contract64.cu, FP64): halfspace counts equal the FP64 oracle's
    outside the tie zone (here: everywhere, the FP64 path has no slack to use),
    projection / asymmetric depths within DEPTH_RTOL, and a short RRS run whose
    halfspace depths equal the oracle's RRS (reference: _kernels.pyx:139-155,
    no dimension limit)."""
    from oracle import oracle
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    n = 5000
    X = toeplitz_gaussian(d, n, seed=4)
    rng = np.random.default_rng(d)
    U = rng.standard_normal((96, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    z = X[11] + 0.05 * rng.standard_normal(d)
    _, cle, cge = b200.evaluate_directions_counts(z, data, U)
    y = X @ U.T - (U @ z)[None, :]
    T = tie_zone(X, z, U)
    assert np.all(np.abs(cle - (y <= 0).sum(axis=0)) <= T) and np.all(np.abs(cge - (y >= 0).sum(axis=0)) <= T)
    ref_h = oracle.evaluate_directions(z, X, U, "halfspace")
    np.testing.assert_array_equal(b200.evaluate_directions(z, data, U, "halfspace", b200.ParallelConfig()), ref_h)
    for notion in ("projection", "asym_projection"):
        got = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig())
        np.testing.assert_allclose(got, oracle.evaluate_directions(z, X, U, notion), rtol=DEPTH_RTOL, atol=0)
    cfg = b200.RrsConfig(total_directions=600, refinements=3, shrink=0.9, notion="halfspace", seed=7)
    Z = np.vstack([X[:3], 0.2 * X[3:5]])
    dg = b200.depth_batch_arrays(Z, data, cfg)[0]
    dr = oracle.depth_batch(Z, X, total_directions=600, refinements=3, shrink=0.9, notion="halfspace", seed=7)[0]
    assert np.array_equal(dg, dr), (dg, dr)


@pytest.mark.parametrize("case", ["tensor_d50", "tensor_d80", "tensor_d200", "convert_d120", "ffma_small_n",
                                  "wide_d300", "ffma_forced"])
def test_early_exit_bitwise(b200, case):
    """RrsConfig(early_exit=True): a query stops once its best count equals the
    rows coinciding with it (the strict-< update, optimizer.py:202, can never
    fire again).  Depth, argmin, min count and every trace record must be
    bitwise those of the full run, for in-sample queries (bound 1, reached
    early), duplicated rows (bound 2), off-sample and far queries (bound 0)."""
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    n, d, path = {"tensor_d50": (20000, 50, "auto"), "tensor_d80": (8000, 80, "auto"),
                  "tensor_d200": (6000, 200, "auto"), "convert_d120": (6000, 120, "convert"),
                  "ffma_small_n": (3000, 6, "auto"), "wide_d300": (3000, 300, "auto"),
                  "ffma_forced": (6000, 12, "ffma")}[case]
    X = toeplitz_gaussian(d, n, seed=9)
    X[1] = X[0]  # a duplicated row: its count bound is 2
    Z = np.vstack([X[:40], 0.3 * X[40:48], X[50:52] * 50.0])
    data = b200.Dataset(X)
    kw = dict(total_directions=3000, refinements=15, shrink=0.8, notion="halfspace", seed=3)
    eng = b200.engine()
    eng.set_contract_path(path)
    try:
        full = b200.depth_batch_arrays(Z, data, b200.RrsConfig(**kw), trace=True)
        eng.enable_timing(True)
        fast = b200.depth_batch_arrays(Z, data, b200.RrsConfig(early_exit=True, **kw), trace=True)
        launches = eng.stats()["kernel_launches"]
        eng.enable_timing(False)
    finally:
        eng.set_contract_path("auto")
    for a, b in zip(full, fast):
        assert np.array_equal(a, b)
    assert full[3][0] >= 2 and full[3][1] >= 2  # the duplicated pair: bound 2
    print(f"\n{case}: final counts {np.bincount(full[3])[:4]}, launches {launches}")


@pytest.mark.parametrize("d", [40, 80])
def test_heterogeneous_columns_projection(b200, d):
    """Columns on scales 1e-3 .. 1e3 and axis-aligned directions: the FP16-split
    tensor stores resolve a point only relative to its largest coordinate, so
    auto must take the FFMA store here (column IQR ratio gate) and every
    per-direction depth must stay within DEPTH_RTOL of the FP64 oracle."""
    from oracle import oracle
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    n = 6000
    X = toeplitz_gaussian(d, n, seed=8) * np.logspace(-3, 3, d)[None, :]
    rng = np.random.default_rng(d)
    U = np.vstack([np.eye(d)[:4], -np.eye(d)[d - 2:], rng.standard_normal((12, d))])
    U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    for notion in ("projection", "asym_projection"):
        for z in (X[4], np.median(X, axis=0)):
            got = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig())
            np.testing.assert_allclose(got, oracle.evaluate_directions(z, X, U, notion), rtol=DEPTH_RTOL, atol=0)
