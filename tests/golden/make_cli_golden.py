"""Golden outputs of the REAL reference CLI (`depthforge depth`, cli.py:113-171)
on committed DFMX / CSV files (docs/formats.md:7-25).

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/{data.dfmx, data.csv, queries.csv} (Toeplitz Gaussian,
n = 600, d = 4; 5 queries: 3 data rows, the origin, a far point) and one JSON
per command: the exact stdout of `depthforge.cli.main([...])` run through the
compiled reference here.  tests/test_io_cli.py replays the same argument lists
through paper_2506_08262_b200.cli on the GPU and compares field by field.
"""

from __future__ import annotations

import contextlib
import io as _io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

OUT = os.path.join(HERE, "cli")

# (name, argv after "depth"); paths are relative to tests/golden/cli
COMMANDS = [
    ("halfspace_dfmx", ["--data", "data.dfmx", "--query", "queries.csv", "--notion", "halfspace",
                        "--k", "2000", "--r", "10", "--seed", "3", "--trace"]),
    ("projection_csv", ["--data", "data.csv", "--query", "queries.csv", "--notion", "projection",
                        "--k", "2000", "--r", "10", "--seed", "3", "--trace"]),
    ("asymprojection_dfmx", ["--data", "data.dfmx", "--query", "queries.csv", "--notion", "asymprojection",
                             "--k", "1000", "--r", "8", "--alpha", "0.8", "--seed", "4"]),
    ("halfspace_inline", ["--data", "data.dfmx", "--query-inline", "0.1,-0.2,0.3,0.05", "--notion", "halfspace",
                          "--k", "3000", "--r", "15", "--seed", "5"]),
    ("mahalanobis_csv", ["--data", "data.csv", "--query", "queries.csv", "--notion", "mahalanobis"]),
]


def write_inputs(df) -> None:
    from depthforge import io as rio
    from depthforge.study.synthetic import ToeplitzGaussianSpec, gen_toeplitz_gaussian

    os.makedirs(OUT, exist_ok=True)
    X = gen_toeplitz_gaussian(ToeplitzGaussianSpec(dim=4, n=600, seed=0))
    Q = np.vstack([X[:3], np.zeros((1, 4)), np.full((1, 4), 6.0)])
    rio.write_matrix(os.path.join(OUT, "data.dfmx"), X)
    rio.write_matrix(os.path.join(OUT, "data.csv"), X)
    rio.write_matrix(os.path.join(OUT, "queries.csv"), Q)


def main() -> None:
    df = import_reference()
    from depthforge import cli as rcli

    write_inputs(df)
    cwd = os.getcwd()
    os.chdir(OUT)
    try:
        for name, argv in COMMANDS:
            buf = _io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = rcli.main(["depth", *argv])
            assert rc == 0, (name, rc)
            payload = json.loads(buf.getvalue())
            with open(f"{name}.json", "w") as fh:
                json.dump({"argv": ["depth", *argv], "stdout": payload}, fh, indent=1, sort_keys=True)
            print(name, "ok")
    finally:
        os.chdir(cwd)


if __name__ == "__main__":
    main()
