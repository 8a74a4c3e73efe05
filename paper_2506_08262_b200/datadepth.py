"""data-depth-style entry points (north_star API):

    halfspace(x, data, NRandom=1000, n_refinements=10, sphcap_shrink=0.5,
              solver="refinedrandom", seed=0)
    projection(...)   aprojection(...)

Mapping onto the reference's RRS: NRandom = total_directions
k (the paper's total over all refinements), n_refinements = r,
sphcap_shrink = alpha, "aprojection" = notion "asym_projection".  Query i of x
uses the Philox substream of index i, exactly like depth_batch
(optimizer.py:254-279).  solver="simplerandom" is RRS with one refinement
(optimizer.py:229-240).
"""

from __future__ import annotations

import numpy as np

from .config import Dataset, DimensionMismatch, RrsConfig
from .solver import depth_batch_arrays

SOLVERS = ("refinedrandom", "simplerandom")


def _run(notion, x, data, NRandom, n_refinements, sphcap_shrink, solver, seed, output_option):
    if solver not in SOLVERS:
        raise ValueError(f"solver {solver!r} is not available on the B200 RRS path (use one of {SOLVERS})")
    ds = data if isinstance(data, Dataset) else Dataset(data)
    X = np.ascontiguousarray(x, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    if X.shape[1] != ds.dim:
        raise DimensionMismatch(f"query dimension {X.shape[1]} does not match data dimension {ds.dim}")
    r = 1 if solver == "simplerandom" else int(n_refinements)
    shrink = 0.5 if solver == "simplerandom" else float(sphcap_shrink)
    cfg = RrsConfig(total_directions=int(NRandom), refinements=r, shrink=shrink, notion=notion,
                    seed=int(seed))
    depth, argmin, _, _ = depth_batch_arrays(X, ds, cfg)
    if output_option == "lowest_depth":
        return depth
    if output_option == "final_direction":
        return depth, argmin
    raise ValueError("output_option must be 'lowest_depth' or 'final_direction'")


def halfspace(x, data, NRandom=1000, n_refinements=10, sphcap_shrink=0.5, solver="refinedrandom",
              seed=0, output_option="lowest_depth"):
    return _run("halfspace", x, data, NRandom, n_refinements, sphcap_shrink, solver, seed, output_option)


def projection(x, data, NRandom=1000, n_refinements=10, sphcap_shrink=0.5, solver="refinedrandom",
               seed=0, output_option="lowest_depth"):
    return _run("projection", x, data, NRandom, n_refinements, sphcap_shrink, solver, seed, output_option)


def aprojection(x, data, NRandom=1000, n_refinements=10, sphcap_shrink=0.5, solver="refinedrandom",
                seed=0, output_option="lowest_depth"):
    return _run("asym_projection", x, data, NRandom, n_refinements, sphcap_shrink, solver, seed,
                output_option)
