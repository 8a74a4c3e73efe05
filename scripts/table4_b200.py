"""The paper's Table 4 at full scale on one B200: Kendall
tau / Spearman rho between the true density ordering and D_P / D_AP (RRS,
k = 1e5, r = 40, alpha = 0.9), n = 1e5 Toeplitz-Gaussian points, 5000
in-sample queries, d in {5, 50, 150}, plus the Mahalanobis baseline.

    python scripts/table4_b200.py --out gpurun_out/table4.json [--queries 5000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_08262_b200 as rrs  # noqa: E402
from paper_2506_08262_b200 import study  # noqa: E402

PAPER = {5: {"projection": 0.9929, "asym_projection": 0.9697}, 50: {"projection": 0.9687, "asym_projection": 0.8820},
         150: {"projection": 0.9216, "asym_projection": 0.7468}}

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/table4.json")
ap.add_argument("--queries", type=int, default=5000)
ap.add_argument("--dims", default="5,50,150")
a = ap.parse_args()
res = {"settings": {"n": 100_000, "k": 100_000, "r": 40, "alpha": 0.9, "queries": a.queries, "seed": 0},
       "paper_kendall": PAPER, "rows": []}
for d in [int(v) for v in a.dims.split(",")]:
    t0 = time.time()
    cfg = rrs.RrsConfig(total_directions=100_000, refinements=40, shrink=0.9, seed=0)
    rs = study.rank_study(study.ToeplitzGaussianSpec(dim=d, n=100_000, seed=0), ["projection", "asym_projection"],
                          a.queries, cfg)
    dt = time.time() - t0
    for row in rs.rows:
        res["rows"].append(dict(row, seconds=dt))
    print(d, round(dt, 1), [(r["pair"], round(r["kendall"], 4)) for r in rs.rows], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
