"""One projection-depth evaluation at a long-row shape, for ncu captures of the
select kernel (scripts/gpu_prof_sel.sh): n points, d = 8, m directions."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as rrs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--m", type=int, default=2048)
ap.add_argument("--notion", default="projection")
ap.add_argument("--select", default="auto")
args = ap.parse_args()
rng = np.random.default_rng(1)
X = rng.standard_normal((args.n, 8))
U = rng.standard_normal((args.m, 8))
U /= np.linalg.norm(U, axis=1)[:, None]
rrs.load_library()
rrs.engine().set_select_path(args.select)
data = rrs.Dataset(X)
for _ in range(2):
    d = rrs.evaluate_directions(X[3], data, U, args.notion, rrs.ParallelConfig(workers=1))
print("mean depth", float(np.mean(d)))
