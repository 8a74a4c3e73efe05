"""Matrix files (DFMX / CSV, docs/formats.md) and the command line.  CPU-only
except the end-to-end depth command, which needs the device."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2506_08262_b200 import cli, io


def test_dfmx_layout_and_round_trip(tmp_path):
    x = np.random.default_rng(0).standard_normal((7, 3))
    p = tmp_path / "x.dfmx"
    io.write_matrix(p, x)
    raw = p.read_bytes()
    assert raw[:4] == b"DFMX" and struct.unpack("<QQ", raw[4:20]) == (7, 3) and len(raw) == 20 + 8 * 21
    assert np.array_equal(np.frombuffer(raw, "<f8", offset=20).reshape(7, 3), x)
    assert np.array_equal(io.read_matrix(p), x)


def test_csv_round_trip_is_exact(tmp_path):
    x = np.random.default_rng(1).standard_normal((5, 4)) * 1e-7 + 1.0 / 3.0
    p = tmp_path / "x.csv"
    io.write_matrix(p, x)
    assert p.read_text().splitlines()[0] == "x0,x1,x2,x3"
    assert np.array_equal(io.read_matrix(p), x)
    io.write_matrix_csv(p, x, header=False)
    assert np.array_equal(io.read_matrix(p), x)


@pytest.mark.parametrize("content,msg", [
    (b"DFMX" + struct.pack("<QQ", 2, 2) + b"\0" * 8, "header implies"),
    (b"DFMX\0\0", "truncated"),
    (b"a,b\n1,2\n3\n", "columns"),
    (b"1,2\nx,y\n", "not numeric"),
    (b"a,b\n", "no data rows"),
    (b"1,nan\n", "non-finite"),
])
def test_malformed_files(tmp_path, content, msg):
    p = tmp_path / "bad"
    p.write_bytes(content)
    with pytest.raises(io.MatrixFormatError, match=msg):
        io.read_matrix(p)
    with pytest.raises(io.MatrixFormatError, match="no such file"):
        io.read_matrix(tmp_path / "missing")


def test_cli_exit_codes(tmp_path, capsys):
    x = tmp_path / "x.dfmx"
    io.write_matrix(x, np.random.default_rng(2).standard_normal((10, 3)))
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3\n")
    assert cli.main(["depth", "--data", str(x), "--query-inline", "1,2", "--notion", "halfspace"]) == cli.EXIT_DIM_MISMATCH
    assert "does not match data dimension 3" in capsys.readouterr().err
    assert cli.main(["depth", "--data", str(bad), "--query-inline", "1", "--notion", "halfspace"]) == cli.EXIT_BAD_DATA
    assert cli.main(["depth", "--data", str(x), "--query-inline", "1,a,2", "--notion", "projection"]) == cli.EXIT_BAD_DATA
    assert cli.main(["depth", "--data", str(x), "--query-inline", "1,2,3", "--notion", "halfspace",
                     "--k", "5", "--r", "10"]) == cli.EXIT_BAD_FLAGS  # RrsConfig: k < r
    assert cli.main(["depth", "--data", str(x)]) == 2  # argparse usage error


def test_cli_gen(tmp_path):
    out = tmp_path / "g.dfmx"
    assert cli.main(["gen", "--dist", "student", "--nu", "1", "--d", "4", "--n", "50", "--seed", "3", "--out", str(out)]) == 0
    from paper_2506_08262_b200.synthetic import student_t

    assert np.array_equal(io.read_matrix(out), student_t(4, 50, 1.0, seed=3))
    assert cli.main(["gen", "--dist", "student", "--d", "4", "--n", "5", "--out", str(out)]) == cli.EXIT_BAD_FLAGS
    assert cli.main(["gen", "--dist", "exponential", "--d", "2", "--n", "6", "--seed", "9", "--out", str(out)]) == 0
    from paper_2506_08262_b200.study import ExponentialSpec, generate

    assert np.array_equal(io.read_matrix(out), generate(ExponentialSpec(dim=2, n=6, seed=9)))


def test_cli_mahalanobis_depth(tmp_path, capsys):
    """Host algebra, no device: (1 + quadratic form)^-1 with the MLE estimate."""
    from paper_2506_08262_b200 import estimate_mle, mahalanobis_depth_batch

    X = np.random.default_rng(3).standard_normal((40, 3))
    io.write_matrix(tmp_path / "x.dfmx", X)
    capsys.readouterr()
    assert cli.main(["depth", "--data", str(tmp_path / "x.dfmx"), "--query-inline", "0.1,0.2,0.3",
                     "--notion", "mahalanobis"]) == 0
    out = json.loads(capsys.readouterr().out)
    want = mahalanobis_depth_batch(np.array([[0.1, 0.2, 0.3]]), estimate_mle(X))[0]
    assert out["backend"] == "b200" and out["query_count"] == 1 and out["results"] == [{"depth": float(want)}]


def test_rows_csv_and_config(tmp_path):
    rows = [{"a": 1, "b": 1.0 / 3.0, "c": "x"}, {"a": 2, "b": 2.5, "c": "y"}]
    io.write_rows_csv(tmp_path / "r.csv", rows)
    back = io.read_rows_csv(tmp_path / "r.csv")
    assert back[0] == {"a": "1", "b": "0.33333333333333331", "c": "x"} and float(back[0]["b"]) == 1.0 / 3.0
    (tmp_path / "c.cfg").write_text("# comment\nalphas = 0.6, 0.9  # trailing\n\nqueries=5\n")
    assert io.parse_config(tmp_path / "c.cfg") == {"alphas": "0.6, 0.9", "queries": "5"}
    assert io.parse_list("1, 2,,3", int) == [1, 2, 3]
    (tmp_path / "bad.cfg").write_text("novalue\n")
    with pytest.raises(ValueError, match="key = value"):
        io.parse_config(tmp_path / "bad.cfg")


def test_cli_fit_model(tmp_path, capsys):
    """fit-model on breakdown-style rows: constants recovered, --predict plateau,
    exit 3 for missing columns, exit 6 for a rank-deficient design."""
    from paper_2506_08262_b200 import perfmodel as pm
    from paper_2506_08262_b200.study import profile_rows

    C = pm.CostConstants(c_const=1e-3, c_rv=1e-9, c_proj=1e-12, c_depth=2e-11)
    profs = []
    for n, d, k, r in ((1000, 5, 400, 2), (5000, 10, 900, 3), (20000, 3, 2000, 4), (8000, 40, 600, 1), (3000, 7, 5000, 5)):
        w = pm.Workload(n=n, d=d, k=k, r=r, g=148, lam=1.5, d_chunk=1)
        g, p, u = pm._terms(w, "parallel")
        profs.append(pm.TimingProfile(workload=w, generation=C.c_rv * g, projection=C.c_proj * p,
                                      univariate=C.c_depth * u, total=C.c_const + C.c_rv * g + C.c_proj * p
                                      + C.c_depth * u, path="parallel"))
    io.write_rows_csv(tmp_path / "b.csv", profile_rows(profs))
    capsys.readouterr()
    assert cli.main(["fit-model", "--profiles", str(tmp_path / "b.csv"), "--predict", "--g", "148",
                     "--lambda", "1.5", "--d", "50", "--d-chunk", "1"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["constants"]["c_proj"] == pytest.approx(1e-12, rel=1e-9)
    assert out["predict"]["plateau"] == pytest.approx(pm.speedup_plateau(C, 50, 1, 148, 1.5), rel=1e-6)
    io.write_rows_csv(tmp_path / "short.csv", [{"n": 1, "d": 2}])
    assert cli.main(["fit-model", "--profiles", str(tmp_path / "short.csv")]) == cli.EXIT_BAD_DATA
    io.write_rows_csv(tmp_path / "same.csv", profile_rows([profs[0]] * 4))
    assert cli.main(["fit-model", "--profiles", str(tmp_path / "same.csv")]) == cli.EXIT_RANK_DEFICIENT
    assert cli.main(["study", "rank", "--out", str(tmp_path / "f" / "x"), "--dist", "student", "--d", "3"]) \
        == cli.EXIT_BAD_FLAGS   # --nu required, checked before any device work


@pytest.mark.gpu
def test_cli_depth_matches_api(b200, tmp_path, capsys):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((500, 4))
    io.write_matrix(tmp_path / "x.dfmx", X)
    io.write_matrix(tmp_path / "q.csv", X[:3])
    rc = cli.main(["depth", "--data", str(tmp_path / "x.dfmx"), "--query", str(tmp_path / "q.csv"),
                   "--notion", "asymprojection", "--k", "200", "--r", "5", "--seed", "9", "--trace"])
    assert rc == 0
    out = json.loads(capsys.readouterr().out)
    cfg = b200.RrsConfig(total_directions=200, refinements=5, shrink=0.9, notion="asym_projection", seed=9)
    ref = b200.depth_batch(list(X[:3]), b200.Dataset(X), cfg)
    assert out["backend"] == "b200" and out["query_count"] == 3
    for got, want in zip(out["results"], ref):
        assert got["depth"] == want.depth and got["directions_used"] == want.directions_used
        assert np.array_equal(got["argmin_direction"], want.argmin_direction)
        assert len(got["trace"]) == 5 and got["trace"][0]["epsilon"] == want.trace[0].epsilon


GOLD_CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["halfspace_dfmx", "projection_csv", "asymprojection_dfmx", "halfspace_inline",
                                  "mahalanobis_csv"])
def test_cli_depth_matches_reference_golden(b200, name, capsys, monkeypatch):
    """`depth` replayed on the files and argument lists the REAL reference CLI
    was run on (tests/golden/make_cli_golden.py, cli.py:113-171): same payload
    keys and header fields, halfspace depths / traces identical, projection
    notions within the tier-2 tolerance, argmin directions to 1e-12."""
    with open(os.path.join(GOLD_CLI, f"{name}.json")) as fh:
        gold = json.load(fh)
    monkeypatch.chdir(GOLD_CLI)
    assert cli.main(gold["argv"]) == 0
    got, want = json.loads(capsys.readouterr().out), gold["stdout"]
    assert set(got) == set(want)
    assert want["backend"] == "compiled" and got["backend"] == "b200"
    for key in set(want) - {"backend", "results"}:
        assert got[key] == want[key], key
    exact = want["notion"] == "halfspace"
    for g, w in zip(got["results"], want["results"], strict=True):
        assert set(g) == set(w)
        if want["notion"] == "mahalanobis":
            assert g["depth"] == pytest.approx(w["depth"], rel=1e-12)
            continue
        if exact:
            assert g["depth"] == w["depth"]
        else:
            assert g["depth"] == pytest.approx(w["depth"], rel=1e-5)
        assert g["directions_used"] == w["directions_used"]
        np.testing.assert_allclose(g["argmin_direction"], w["argmin_direction"], rtol=0, atol=1e-12)
        if "trace" in w:
            assert len(g["trace"]) == len(w["trace"])
            for gt, wt in zip(g["trace"], w["trace"]):
                assert gt["epsilon"] == wt["epsilon"]
                if exact:
                    assert gt["best_depth"] == wt["best_depth"]
                else:
                    assert gt["best_depth"] == pytest.approx(wt["best_depth"], rel=1e-5)
                np.testing.assert_allclose(gt["pole"], wt["pole"], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_read_matrix_pinned(b200, tmp_path):
    """read_matrix(..., pinned=True): same values as the pageable read, in
    page-locked memory (DFMX read straight into it, CSV copied once)."""
    import torch

    X = np.random.default_rng(8).standard_normal((3001, 7))
    for fname in ("x.dfmx", "x.csv"):
        io.write_matrix(tmp_path / fname, X)
        a = io.read_matrix(tmp_path / fname)
        p = io.read_matrix(tmp_path / fname, pinned=True)
        assert np.array_equal(a, p) and np.array_equal(p, X)
        assert torch.from_numpy(p).is_pinned()
        data = b200.Dataset(p)
        cfg = b200.RrsConfig(total_directions=300, refinements=3, shrink=0.9, notion="halfspace", seed=2)
        assert np.array_equal(b200.depth_batch_arrays(p[:4], data, cfg)[0],
                              b200.depth_batch_arrays(a[:4], b200.Dataset(a), cfg)[0])
    (tmp_path / "bad.dfmx").write_bytes((tmp_path / "x.dfmx").read_bytes()[:-8])
    with pytest.raises(io.MatrixFormatError):
        io.read_matrix(tmp_path / "bad.dfmx", pinned=True)
