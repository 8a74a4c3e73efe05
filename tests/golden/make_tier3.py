"""Tier-3 fixtures at the BASELINE.json shapes, from the REAL reference.

    python tests/golden/make_tier3.py c2 c3 c4      # ~10 min on 8 cores
    python tests/golden/make_tier3.py c5h c5p       # ~1 h (n = 1M, d = 200)

Runs the reference's compiled ``depth_batch`` (optimizer.py:254-279; query i on
substream i) at k = 20,000, r = 20, alpha = 0.9, seed = 1 on the datasets and
query sets of tests/golden/tier3_data.py, and writes
tests/golden/tier3_<tag>.npz with the depths, argmin directions and the trace
of best depths.  Config 5 runs one query at a time through
``refined_random_search(..., query_index=i)`` with all cores inside the query
(px is 8 GB per concurrent query there), which the reference
documents as bit-identical to ``depth_batch`` element i.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import tier3_data as T  # noqa: E402
from make_golden import import_reference  # noqa: E402


def run(tag: str, df) -> None:
    notion, n, d, dist, k, r, alpha = T.CASES[tag]
    X = T.dataset(tag)
    Z = T.queries(tag, X)
    workers = os.cpu_count()
    data = df.Dataset(X)
    t0 = time.time()
    if n >= 1_000_000:
        cfg = df.RrsConfig(total_directions=k, refinements=r, shrink=alpha, notion=notion, seed=1,
                           parallel=df.ParallelConfig(workers=workers))
        res = []
        for i, z in enumerate(Z):
            res.append(df.refined_random_search(z, data, cfg, query_index=i))
            print(f"  {tag} query {i}: depth {res[-1].depth:.8g} ({time.time() - t0:.0f} s)", flush=True)
    else:
        cfg = df.RrsConfig(total_directions=k, refinements=r, shrink=alpha, notion=notion, seed=1,
                           parallel=df.ParallelConfig(workers=workers))
        res = df.depth_batch(list(Z), data, cfg)
    dt = time.time() - t0
    out = {
        "args": np.array([n, d, k, r], dtype=np.int64),
        "alpha": np.array(alpha),
        "notion": np.array(notion),
        "dist": np.array(dist),
        "x_digest": np.array(T.digest(X)),
        "z": Z,
        "depth": np.array([x.depth for x in res]),
        "argmin": np.stack([x.argmin_direction for x in res]),
        "trace_best": np.array([[t.best_depth for t in x.trace] for x in res]),
        "seconds": np.array(dt),
        "workers": np.array(workers),
    }
    path = os.path.join(HERE, f"tier3_{tag}.npz")
    np.savez_compressed(path, **out)
    print(f"{tag}: {len(res)} queries in {dt:.0f} s on {workers} cores -> {path}", flush=True)


def main(argv):
    df = import_reference()
    for tag in argv or ["c2", "c3", "c4"]:
        run(tag, df)


if __name__ == "__main__":
    main(sys.argv[1:])
