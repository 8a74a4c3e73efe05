"""Study drivers on one B200:

1. phase breakdown (CUDA-event phases) over a workload set + the paper's T_G
   fit with measured lam = f_CPU / f_GPU (host "cpu MHz" / SM clock sampled
   by nvidia-smi during the runs), g = 148 SMs;
2. rank study (pdf ordering vs RRS depths, Spearman / Kendall) at the
   reference CLI's --full settings (500 of the 5000 queries);
3. convergence frontier (minimal r per (d, k)) at the reference CLI's --full
   settings (the paper's Table 4 grid);
4. the paper's published D_P timing tables (Tables 1 and 3) re-run.

    python scripts/study_b200.py --out gpurun_out/study.json
"""

import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08262_b200 as rrs  # noqa: E402
from paper_2506_08262_b200 import perfmodel as pm  # noqa: E402
from paper_2506_08262_b200 import study  # noqa: E402


def cpu_mhz() -> float:
    vals = [float(l.split(":")[1]) for l in open("/proc/cpuinfo") if l.startswith("cpu MHz")]
    return float(np.median(vals)) if vals else float("nan")


def sm_mhz() -> float:
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout
        return float(out.split()[0])
    except Exception:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/study.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="", help="comma list of sections to run (breakdown,rank,frontier,tables)")
    a = ap.parse_args()
    res = {}
    only = {x for x in a.only.split(",") if x}

    def want(section: str) -> bool:
        return not only or section in only

    if want("breakdown"):
        # 1. breakdown + fit ---------------------------------------------------
        shapes = [(20_000, 10, 2_000, 2), (50_000, 20, 4_000, 4), (100_000, 50, 10_000, 10), (100_000, 50, 20_000, 20),
                  (30_000, 50, 6_000, 3), (200_000, 8, 3_000, 3), (60_000, 100, 2_000, 2), (10_000, 20, 20_000, 20)]
        if a.quick:
            shapes = shapes[:4]
        clocks = []
        for notion in ("halfspace", "projection"):
            prof_f = []
            f_cpu = cpu_mhz()
            t0 = time.time()
            ws0 = [pm.Workload(n=n, d=d, k=k, r=r, g=148, lam=1.0, d_chunk=1) for n, d, k, r in shapes]
            study.breakdown_bench(ws0[:1], notion, "parallel", repeats=1)          # warm the library + dataset path
            clocks.append(sm_mhz())
            profs = study.breakdown_bench(ws0, notion, "parallel", repeats=5)
            clocks.append(sm_mhz())
            f_gpu = float(np.nanmax(clocks)) if np.isfinite(clocks).any() else float("nan")
            lam = f_cpu / f_gpu if np.isfinite(f_cpu) and np.isfinite(f_gpu) and f_gpu > 0 else 1.0
            # re-label the workloads with the measured lam (phase times unchanged)
            for p in profs:
                w = p.workload
                prof_f.append(pm.TimingProfile(workload=pm.Workload(n=w.n, d=w.d, k=w.k, r=w.r, g=148, lam=lam,
                                                                    d_chunk=1),
                                               generation=p.generation, projection=p.projection,
                                               univariate=p.univariate, total=p.total, path="parallel"))
            rep = pm.fit_constants(prof_f)
            pred = [pm.t_parallel(rep.constants, p.workload) for p in prof_f]
            res[f"breakdown_{notion}"] = {
                "f_cpu_mhz": f_cpu, "f_gpu_mhz": f_gpu, "lam": lam, "g": 148, "d_chunk": 1,
                "rows": study.profile_rows(prof_f),
                "fit": json.loads(rep.to_json()),
                "predicted_total_s": pred, "measured_total_s": [p.total for p in prof_f],
                "seconds": time.time() - t0,
            }
            print(notion, "fit", rep.to_json().replace("\n", " ")[:400], flush=True)

    if want("rank"):
        # 2. rank study: the reference CLI's --full settings (d = 50, n = 100k, k = 100k,
        #    r = 40, projection + asym_projection) on a bounded number of queries
        from paper_2506_08262_b200.cli import STUDY_SETTINGS

        full = STUDY_SETTINGS["rank"][1]
        t0 = time.time()
        spec = study.ToeplitzGaussianSpec(dim=int(full["d"]), n=int(full["n"]), seed=0)
        cfg = rrs.RrsConfig(total_directions=int(full["k"]), refinements=int(full["r"]), shrink=float(full["alpha"]),
                            seed=0)
        nq = 100 if a.quick else 500
        rs = study.rank_study(spec, full["notions"].split(","), nq, cfg)
        res["rank_study_full_settings"] = {"settings": dict(full, queries=str(nq)), "rows": list(rs.rows),
                                           "seconds": time.time() - t0}
        print("rank", rs.rows, time.time() - t0, flush=True)

    if want("frontier"):
        # 3. convergence frontier: the reference CLI's --full settings (Table 4 grid:
        #    d in 5..175, k up to 1e5, r up to 175, reference k = 3e5 x 3 repeats)
        fs = STUDY_SETTINGS["frontier"][1]
        t0 = time.time()
        dims = [int(v) for v in fs["dims"].split(",")]
        grid = study.StudyGrid(alphas=(float(fs["alphas"]),),
                               refinement_counts=tuple(int(v) for v in fs["refinements"].split(",")),
                               direction_counts=tuple(int(v) for v in fs["directions"].split(",")),
                               dims=tuple(dims[:2] if a.quick else dims), query_count=int(fs["queries"]),
                               reference=study.ReferenceSpec(k=int(fs["ref_k"]), r=int(fs["ref_r"]),
                                                            alpha=float(fs["ref_alpha"]), repeats=int(fs["ref_repeats"])))
        fr = study.convergence_frontier(grid, fs["notion"], study.ToeplitzGaussianSpec(dim=dims[0], n=int(fs["n"]), seed=0),
                                        tol=float(fs["tol"]), seed=0)
        res["frontier_full_settings"] = {"settings": fs, "rows": list(fr.rows), "seconds": time.time() - t0}
        print("frontier", fr.rows, time.time() - t0, flush=True)

    if want("tables"):
        # 4. the paper's published D_P timing tables (RTX 4080 laptop GPU, seconds per
        #    query point) re-run on the B200 with runtime_grid:
        #    Table 1 (n = 10k, r = 1, k = 1e4 / 1e5 / 2.5e5, d = 5..150) and
        #    Table 3 (n = 100k, r = 1, k = 1e4, d = 5..150)
        t0 = time.time()
        dims = (5, 25, 50, 100, 150)
        t1 = study.runtime_grid(dims, (10_000, 100_000, 250_000), n=10_000, r=1, notion="projection", repeats=5)
        t3 = study.runtime_grid(dims, (10_000,), n=100_000, r=1, notion="projection", repeats=5)
        res["paper_tables"] = {"table1_n10k_r1": list(t1.rows), "table3_n100k_r1": list(t3.rows),
                               "paper_rtx4080_s": {"table1_k1e4": 0.03, "table1_k1e5": [0.26, 0.30],
                                                   "table1_k2.5e5": [2.49, 2.66], "table3_k1e4": [0.28, 0.33]},
                               "seconds": time.time() - t0}
        print("paper tables", t1.rows, t3.rows, flush=True)

    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1, default=float)


if __name__ == "__main__":
    main()
