"""Golden fixtures for the study harness and the perfmodel (SURVEY.md §8(f)
rows 3-4) from the REAL reference; build container only:

    python tests/golden/make_study_golden.py

Reuses make_golden.import_reference (the reference's own compiled core in a
scratch copy).  Writes tests/golden/study_golden.npz; every array comes from
the reference call named next to it.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402


def main():
    df = import_reference()
    from depthforge import perfmodel as pm
    from depthforge import study
    from depthforge.univariate import estimate_mle, mahalanobis_depth_batch

    out = {}
    rng = np.random.default_rng(77)

    # --- correlation.py:24-105 on tie-heavy integer vectors + continuous ones
    vecs_a, vecs_b, rho, tau = [], [], [], []
    for i in range(40):
        n = int(rng.integers(2, 300))
        if i % 2:
            a, b = rng.integers(0, 6, n).astype(float), rng.integers(0, 6, n).astype(float)
        else:
            a, b = rng.standard_normal(n), rng.standard_normal(n)
        try:
            r, t = study.spearman_rho(a, b), study.kendall_tau(a, b)
        except ValueError:
            continue
        vecs_a.append(np.pad(a, (0, 300 - n), constant_values=np.nan))
        vecs_b.append(np.pad(b, (0, 300 - n), constant_values=np.nan))
        rho.append(r)
        tau.append(t)
    out["corr_a"], out["corr_b"] = np.array(vecs_a), np.array(vecs_b)
    out["corr_rho"], out["corr_tau"] = np.array(rho), np.array(tau)
    x = rng.integers(0, 9, 500).astype(float)
    out["ranks_in"], out["ranks_out"] = x, study.average_ranks(x)

    # --- synthetic.py:76-144
    spec = study.ToeplitzGaussianSpec(dim=4, n=50, seed=3)
    out["qf_queries"] = study.generate(spec)
    out["qf_out"] = study.quadratic_forms(spec, out["qf_queries"])
    out["exp_sample"] = study.generate(study.ExponentialSpec(dim=3, n=20, seed=9))
    tspec = study.StudentTSpec(dim=3, n=30, nu=2.5, seed=4)
    out["t_sample"] = study.generate(tspec)
    out["t_density_rank"] = study.true_density_rank(tspec, out["t_sample"])
    out["maha_out"] = mahalanobis_depth_batch(out["t_sample"][:10], estimate_mle(out["t_sample"]))

    # --- perfmodel.py:102-261
    W = [dict(n=1000 + 37 * i, d=3 + i % 7, k=200 + 50 * i, r=1 + i % 5, g=1 + 3 * i, lam=0.5 + 0.1 * i,
              d_chunk=1 + i % 4) for i in range(12)]
    C = pm.CostConstants(c_const=0.01, c_rv=2e-9, c_proj=3e-10, c_depth=5e-9)
    out["pm_workloads"] = json.dumps(W)
    out["pm_tseq"] = np.array([pm.t_sequential(C, pm.Workload(**w)) for w in W])
    out["pm_tpar"] = np.array([pm.t_parallel(C, pm.Workload(**w)) for w in W])
    out["pm_speedup"] = np.array([pm.speedup(C, pm.Workload(**w)) for w in W])
    out["pm_plateau"] = np.array([pm.speedup_plateau(C, 50, 8, 148, 1.7), pm.speedup_plateau(C, 7, 256, 16, 1.0)])
    noise = rng.uniform(0.9, 1.1, size=(12, 3))
    profs = []
    for i, w in enumerate(W):
        wl = pm.Workload(**w)
        path = "sequential" if i < 6 else "parallel"
        seq = path == "sequential"
        g = wl.r * wl.m * wl.d if seq else wl.r * wl.lam * -(-wl.m * wl.d // wl.g)
        p = wl.r * wl.m * wl.n * wl.d if seq else wl.r * wl.lam * -(-wl.d // wl.d_chunk) * -(-wl.m * wl.n // wl.g)
        u = wl.r * wl.depth_units if seq else wl.r * wl.lam * np.ceil(wl.depth_units / wl.g)
        ph = np.array([C.c_rv * g, C.c_proj * p, C.c_depth * u]) * noise[i]
        profs.append(pm.TimingProfile(workload=wl, generation=ph[0], projection=ph[1], univariate=ph[2],
                                      total=ph.sum() + 0.01 * noise[i, 0], path=path))
    out["pm_profiles"] = json.dumps([dict(w=W[i], g=p.generation, p=p.projection, u=p.univariate, t=p.total,
                                          path=p.path) for i, p in enumerate(profs)])
    rep = pm.fit_constants(profs)
    c = rep.constants
    out["pm_fit"] = np.array([c.c_const, c.c_rv, c.c_proj, c.c_depth, rep.r_squared, rep.max_rel_residual])
    out["pm_fit_residuals"] = np.array(rep.residuals)

    # --- study/rank.py:33-86 (depths by the reference's compiled RRS)
    cfg = df.RrsConfig(total_directions=1000, refinements=5, shrink=0.9, seed=1,
                       parallel=df.ParallelConfig(workers=4))
    res = study.rank_study(study.ToeplitzGaussianSpec(dim=3, n=400, seed=0),
                           ["halfspace", "projection", "asym_projection"], 40, cfg)
    out["rank_rows"] = json.dumps(list(res.rows))
    for k, v in res.depths.items():
        out[f"rank_depth_{k}"] = v

    # --- study/convergence.py:112-221
    grid = study.StudyGrid(alphas=(0.9,), refinement_counts=(2, 4), direction_counts=(100, 200), dims=(3,),
                           query_count=6, reference=study.ReferenceSpec(k=1000, r=5, alpha=0.9, repeats=2))
    data = df.Dataset(study.generate(study.ToeplitzGaussianSpec(dim=3, n=400, seed=0)))
    conv = study.convergence_study(grid, "projection", data, seed=1, workers=4)
    out["conv_refs"] = conv.references
    out["conv_means"] = json.dumps(list(conv.cell_means))
    fr = study.convergence_frontier(grid, "halfspace", study.ToeplitzGaussianSpec(dim=3, n=300, seed=5),
                                    tol=1e-3, seed=2, workers=4)
    out["frontier_rows"] = json.dumps(list(fr.rows))

    np.savez_compressed(os.path.join(HERE, "study_golden.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
