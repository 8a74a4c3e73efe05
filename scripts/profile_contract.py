"""Small driver for ncu captures of the hot kernels (config-4 shape, 64 queries,
2 refinements; or --notion projection for the store + select path)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as rrs  # noqa: E402
from paper_2506_08262_b200.synthetic import toeplitz_gaussian  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--notion", default="halfspace")
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--d", type=int, default=50)
ap.add_argument("--q", type=int, default=1024)
ap.add_argument("--m", type=int, default=1000)
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
rrs.engine().set_contract_path(a.path)
X = toeplitz_gaussian(a.d, a.n, seed=0)
cfg = rrs.RrsConfig(total_directions=a.m * a.r, refinements=a.r, shrink=0.9, notion=a.notion, seed=1)
out = rrs.depth_batch_arrays(X[: a.q], rrs.Dataset(X), cfg)
print("min counts", out[3][:8])
