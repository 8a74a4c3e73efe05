"""Matrix files (DFMX / CSV, docs/formats.md) and the command line.  CPU-only
except the end-to-end depth command, which needs the device."""

import json
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
    assert cli.main(["depth", "--data", str(x), "--query-inline", "1,2,3", "--notion", "mahalanobis"]) == cli.EXIT_BAD_FLAGS
    assert cli.main(["depth", "--data", str(x), "--query-inline", "1,2,3", "--notion", "halfspace",
                     "--k", "5", "--r", "10"]) == cli.EXIT_BAD_FLAGS  # RrsConfig: k < r
    assert cli.main(["depth", "--data", str(x)]) == 2  # argparse usage error


def test_cli_gen(tmp_path):
    out = tmp_path / "g.dfmx"
    assert cli.main(["gen", "--dist", "student", "--nu", "1", "--d", "4", "--n", "50", "--seed", "3", "--out", str(out)]) == 0
    from paper_2506_08262_b200.synthetic import student_t

    assert np.array_equal(io.read_matrix(out), student_t(4, 50, 1.0, seed=3))


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
