"""Study drivers on the B200 engine (rank study,
convergence study / frontier; row 4: phase breakdown) against the reference's
own study outputs (tests/golden/study_golden.npz) and the reference's
test_studies.py cases."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "study_golden.npz"))
DEPTH_RTOL = 1e-5


def _json(key):
    return json.loads(str(GOLD[key]))


def _grid(study, **kw):
    base = dict(alphas=(0.9,), refinement_counts=(2, 4), direction_counts=(100, 200), dims=(3,), query_count=6,
                reference=study.ReferenceSpec(k=1000, r=5, alpha=0.9, repeats=2))
    base.update(kw)
    return study.StudyGrid(**base)


def test_rank_study_matches_reference(b200):
    from paper_2506_08262_b200 import study

    cfg = b200.RrsConfig(total_directions=1000, refinements=5, shrink=0.9, seed=1)
    res = study.rank_study(study.ToeplitzGaussianSpec(dim=3, n=400, seed=0),
                           ["halfspace", "projection", "asym_projection"], 40, cfg)
    np.testing.assert_array_equal(res.depths["halfspace"], GOLD["rank_depth_halfspace"])
    for k in ("projection", "asym_projection"):
        np.testing.assert_allclose(res.depths[k], GOLD[f"rank_depth_{k}"], rtol=DEPTH_RTOL, atol=0)
    np.testing.assert_allclose(res.depths["mahalanobis"], GOLD["rank_depth_mahalanobis"], rtol=1e-13)
    want = _json("rank_rows")
    assert [r["pair"] for r in res.rows] == [r["pair"] for r in want]
    for got, ref in zip(res.rows, want):
        exact = ref["pair"] in ("pdf_x_halfspace", "pdf_x_mahalanobis")
        tol = 1e-12 if exact else 2e-3   # a 1e-5 depth difference may swap one near-tied pair
        assert got["spearman"] == pytest.approx(ref["spearman"], abs=tol)
        assert got["kendall"] == pytest.approx(ref["kendall"], abs=tol)


def test_convergence_study_matches_reference(b200):
    from paper_2506_08262_b200 import study

    grid = _grid(study)
    data = b200.Dataset(study.generate(study.ToeplitzGaussianSpec(dim=3, n=400, seed=0)))
    res = study.convergence_study(grid, "projection", data, seed=1, workers=4)
    np.testing.assert_allclose(res.references, GOLD["conv_refs"], rtol=DEPTH_RTOL, atol=0)
    want = _json("conv_means")
    assert len(res.cell_means) == len(want) == 4
    for got, ref in zip(res.cell_means, want):
        assert {k: got[k] for k in ("alpha", "r", "k", "d")} == {k: ref[k] for k in ("alpha", "r", "k", "d")}
        assert got["mean_mse"] == pytest.approx(ref["mean_mse"], rel=1e-3, abs=1e-9)
    assert len(res.rows) == 4 * grid.query_count
    assert all(set(r) == {"alpha", "r", "k", "d", "point_id", "mse"} and r["mse"] >= 0 for r in res.rows)


def test_frontier_matches_reference(b200):
    from paper_2506_08262_b200 import study

    fr = study.convergence_frontier(_grid(study), "halfspace", study.ToeplitzGaussianSpec(dim=3, n=300, seed=5),
                                    tol=1e-3, seed=2, workers=4)
    assert list(fr.rows) == _json("frontier_rows")


def test_reference_run_reproduces_zero_error(b200):
    from paper_2506_08262_b200 import study
    from paper_2506_08262_b200.study.convergence import _cfg, _pick_queries, reference_depths

    data = b200.Dataset(study.generate(study.ToeplitzGaussianSpec(dim=3, n=400, seed=0)))
    q = _pick_queries(data, 4, 3)
    refs = reference_depths(q, data, "projection", study.ReferenceSpec(k=1000, r=5, alpha=0.9, repeats=1),
                            seed=3, workers=2)
    rerun = np.array([r.depth for r in b200.depth_batch(q, data, _cfg("projection", 1000, 5, 0.9, 3, 2))])
    assert np.array_equal(rerun, refs)


def test_frontier_edge_cases(b200):
    from paper_2506_08262_b200 import study

    grid = _grid(study, dims=(2, 3), query_count=4)
    fr = study.convergence_frontier(grid, "projection", study.ToeplitzGaussianSpec(dim=2, n=300, seed=5),
                                    tol=np.inf, seed=2)
    assert len(fr.rows) == 4
    assert all(r["min_r"] == 2 and r["all_converged"] and r["mean_point_min_r"] == 2 for r in fr.rows)
    one = study.convergence_frontier(_grid(study, query_count=1), "halfspace",
                                     study.ToeplitzGaussianSpec(dim=3, n=1, seed=0), tol=1e-4)
    assert all(r["min_r"] == 2 and r["all_converged"] for r in one.rows)
    expo = study.convergence_frontier(_grid(study, query_count=2, dims=(2,)), "projection",
                                      study.ExponentialSpec(dim=2, n=200, seed=1), tol=np.inf, seed=1)
    assert len(expo.rows) == 2
    with pytest.raises(ValueError, match="single alpha"):
        study.convergence_frontier(_grid(study, alphas=(0.6, 0.9)), "projection",
                                   study.ToeplitzGaussianSpec(dim=3, n=10, seed=0))


def test_breakdown_and_fit(b200):
    """Device phase breakdown (CUDA-event phases, wall total) -> rows -> fit."""
    from paper_2506_08262_b200 import perfmodel as pm
    from paper_2506_08262_b200 import study

    ws = [pm.Workload(n=n, d=d, k=k, r=r, g=148, lam=1.0, d_chunk=1)
          for n, d, k, r in ((2000, 5, 400, 2), (8000, 10, 1200, 3), (4000, 20, 900, 3), (16000, 8, 2000, 4))]
    profs = study.breakdown_bench(ws, "projection", "parallel", seed=0, repeats=3)
    assert len(profs) == 4
    for p in profs:
        assert p.path == "parallel" and p.total >= max(p.generation, p.projection, p.univariate)
        assert min(p.generation, p.projection, p.univariate) > 0
    rows = study.profile_rows(profs)
    for i in range(0, len(rows), 3):
        assert sum(r["fraction"] for r in rows[i:i + 3]) <= 1.0 + 1e-12
    rep = pm.fit_constants(study.profiles_from_rows(rows))
    assert rep.profile_count == 4 and rep.constants.c_proj > 0


def test_runtime_grid(b200):
    from paper_2506_08262_b200 import study

    res = study.runtime_grid((3, 5), (200, 400), n=1000, r=2, notion="halfspace", repeats=2)
    assert len(res.rows) == 4 and all(r["seconds"] > 0 for r in res.rows)


def test_cli_bench_and_study_commands(b200, tmp_path, capsys):
    """The reference's bench / study / fit-model commands end to end on the
    device at desk-test sizes (config files override the desk defaults)."""
    from paper_2506_08262_b200 import cli, io

    cfg = tmp_path / "tiny.cfg"
    cfg.write_text("alphas = 0.9\nrefinements = 2,4\ndirections = 100,200\nd = 3\ndims = 2,3\nn = 300\n"
                   "queries = 4\nref_k = 1000\nref_r = 5\nref_repeats = 1\nk = 500\nr = 5\n"
                   "notions = halfspace,projection\n")
    for cmd, files in ((["study", "converge"], ["converge.csv", "converge_means.csv", "converge_summary.json"]),
                       (["study", "frontier"], ["frontier.csv", "frontier_summary.json"]),
                       (["study", "rank"], ["rank.csv", "rank_summary.json"])):
        out = tmp_path / cmd[1]
        assert cli.main(cmd + ["--config", str(cfg), "--out", str(out), "--seed", "1"]) == 0, cmd
        assert all((out / f).exists() for f in files), cmd
    assert len(io.read_rows_csv(tmp_path / "converge" / "converge.csv")) == 4 * 4
    assert [r["pair"] for r in io.read_rows_csv(tmp_path / "rank" / "rank.csv")] == \
        ["pdf_x_halfspace", "pdf_x_projection", "pdf_x_mahalanobis"]
    bd = tmp_path / "bd"
    assert cli.main(["bench", "breakdown", "--path", "parallel", "--dims", "3,6", "--directions", "200,400",
                     "--n", "2000", "--r", "2", "--repeats", "2", "--workers", "148", "--d-chunk", "1",
                     "--out", str(bd)]) == 0
    assert len(io.read_rows_csv(bd / "breakdown.csv")) == 4 * 3
    capsys.readouterr()
    assert cli.main(["fit-model", "--profiles", str(bd / "breakdown.csv")]) == 0
    assert json.loads(capsys.readouterr().out)["profile_count"] == 4
    assert cli.main(["bench", "grid", "--dims", "3", "--directions", "100,200", "--n", "500", "--repeats", "2",
                     "--notion", "halfspace", "--out", str(tmp_path / "grid")]) == 0
    assert cli.main(["bench", "grid", "--notion", "mahalanobis", "--out", str(tmp_path / "g2")]) == 2
