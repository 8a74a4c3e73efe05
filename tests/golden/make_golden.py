"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch dir, builds the reference's own
Cython core there (`python setup.py build_ext --inplace`, pkg/setup.py:40-59),
imports `depthforge` with DEPTHFORGE_BACKEND=compiled and records its outputs
on seeded inputs.  The fixtures pin (a) the CPU restatement in oracle/ and
(b) the CUDA path, so neither needs the reference at run time.

Every array written here comes from a reference call named next to it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"


def import_reference():
    scratch = os.environ.get("DEPTHFORGE_BUILD_DIR") or os.path.join(tempfile.gettempdir(), "dfref_golden")
    if not os.path.exists(os.path.join(scratch, "src", "depthforge")):
        shutil.rmtree(scratch, ignore_errors=True)
        shutil.copytree(REF, scratch)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=scratch,
                       check=True, stdout=subprocess.DEVNULL)
    os.environ["DEPTHFORGE_BACKEND"] = "compiled"
    sys.path.insert(0, os.path.join(scratch, "src"))
    import depthforge  # noqa: E402

    assert depthforge.backend_name() == "compiled"
    return depthforge


def main():
    df = import_reference()
    from depthforge import philox
    from depthforge.directions import CapSpec, Pole, generate_batch
    from depthforge.projection import project_parallel, project_point
    from depthforge.study.synthetic import (StudentTSpec, ToeplitzGaussianSpec,
                                            gen_student_t, gen_toeplitz_gaussian)
    from scipy.special import ndtri

    out = {}

    # --- Philox / uniforms / ndtri (philox.py:27-125) -----------------------
    rng = np.random.default_rng(2024)
    ctr = rng.integers(0, 2**32, size=(4, 256), dtype=np.uint64).astype(np.uint32)
    out["philox_ctr"] = ctr
    out["philox_key"] = np.array([0x9E3779B9, 0x1234567], dtype=np.uint32)
    out["philox_out"] = philox.philox4x32(ctr, 0x9E3779B9, 0x1234567)
    v = (np.arange(4096) % 51).astype(np.uint32)
    j = np.arange(4096, dtype=np.uint32)
    out["unif_args"] = np.array([123456789123, 7, 4_000_000_001], dtype=np.uint64)  # seed, l, q
    out["unif_v"], out["unif_j"] = v, j
    out["unif_out"] = philox.uniforms(123456789123, v, j, 7, 4_000_000_001)
    y = np.concatenate([out["unif_out"][:2048], rng.uniform(0, 1, 2048),
                        10.0 ** -np.arange(1, 300, 3), 1 - 10.0 ** -np.arange(1, 16)])
    out["ndtri_in"], out["ndtri_out"] = y, ndtri(y)

    # --- numpy pairwise row sums (directions.py:127,162) --------------------
    lens = np.array([1, 2, 7, 8, 9, 15, 16, 17, 49, 50, 127, 128, 129, 199, 200, 257])
    rows = rng.standard_normal((lens.size, 257)) * rng.uniform(0.1, 10, (lens.size, 257))
    out["pw_len"], out["pw_rows"] = lens, rows
    out["pw_out"] = np.array([rows[i, : lens[i]][None, :].sum(axis=1)[0] for i in range(lens.size)])

    # --- cap rows (directions.py:192-204 generate_batch) --------------------
    caps = []
    for idx, (d, m) in enumerate([(1, 5), (2, 33), (5, 100), (9, 40), (50, 64), (200, 16)]):
        for kind in ("e1", "neg_e1", "random"):
            p = np.zeros(d)
            p[0] = 1.0 if kind != "neg_e1" else -1.0
            if kind == "random" and d > 1:
                p = rng.standard_normal(d)
                p /= np.linalg.norm(p)
            eps = float(rng.uniform(0.05, np.pi / 2))
            seed, l, q = int(rng.integers(0, 2**40)), int(rng.integers(0, 40)), int(rng.integers(0, 2**20))
            U = generate_batch(CapSpec(Pole(p), eps), m, seed, refinement=l, query=q).directions
            caps.append((p, eps, m, seed, l, q, U))
    out["cap_count"] = np.array(len(caps))
    for i, (p, eps, m, seed, l, q, U) in enumerate(caps):
        out[f"cap{i}_pole"] = p
        out[f"cap{i}_args"] = np.array([eps, m, seed, l, q], dtype=np.float64)
        out[f"cap{i}_U"] = U

    # --- univariate spans on tie-heavy data (test_backends.py:59-90) --------
    be = df._core.get_backend("compiled")
    for n in (1, 2, 3, 18, 101, 1024):
        r2 = np.random.default_rng(3)
        px = np.round(r2.standard_normal((60, n)) * 4, 1)
        pz = np.round(r2.standard_normal(60) * 4, 1)
        out[f"span_n{n}_px"], out[f"span_n{n}_pz"] = px, pz
        for name in ("halfspace", "projection", "asym_projection"):
            o = np.empty(60)
            getattr(be, f"{name}_span")(px, pz, o, 0, 60)
            out[f"span_n{n}_{name}"] = o
    px = np.array([[2.0, 2.0, 2.0, 2.0], [1.0, 1.0, 1.0, 5.0], [-3.0, -3.0, -1.0, -1.0]])
    pz = np.array([2.0, 6.0, -2.0])
    out["degen_px"], out["degen_pz"] = px, pz
    for name in ("halfspace", "projection", "asym_projection"):
        o = np.empty(3)
        getattr(be, f"{name}_span")(px, pz, o, 0, 3)
        out[f"degen_{name}"] = o

    # --- projection (proj_naive, _kernels.pyx:171-185) ----------------------
    x = rng.standard_normal((41, 13))
    u = rng.standard_normal((29, 13))
    o = np.empty((29, 41))
    be.proj_naive(x, u, o)
    out["proj_x"], out["proj_u"], out["proj_out"] = x, u, o

    # --- evaluate_directions (optimizer.py:98-142), explicit directions -----
    cfgp = df.ParallelConfig(workers=2)
    for tag, (n, d, m, dist) in {"ed_small": (300, 6, 64, "gauss"),
                                 "ed_cauchy": (501, 9, 96, "cauchy")}.items():
        X = (gen_toeplitz_gaussian(ToeplitzGaussianSpec(d, n, seed=4)) if dist == "gauss"
             else gen_student_t(StudentTSpec(d, n, nu=1.0, seed=4)))
        U = rng.standard_normal((m, d))
        U /= np.linalg.norm(U, axis=1)[:, None]
        Z = np.stack([X[0], 0.3 * X[1], np.zeros(d), X[2] + 5.0])
        out[f"{tag}_x"], out[f"{tag}_U"], out[f"{tag}_Z"] = X, U, Z
        for name in ("halfspace", "projection", "asym_projection"):
            res = np.stack([df.evaluate_directions(z, df.Dataset(X), U, name, cfgp) for z in Z])
            out[f"{tag}_{name}"] = res
        pxr = project_parallel(df.Dataset(X), U, cfgp).scores
        cle = np.stack([(pxr <= project_point(z, U)[:, None]).sum(axis=1) for z in Z])
        cge = np.stack([(pxr >= project_point(z, U)[:, None]).sum(axis=1) for z in Z])
        out[f"{tag}_cle"], out[f"{tag}_cge"] = cle, cge

    # --- end-to-end RRS (optimizer.py:254-279) ------------------------------
    # config 1 of BASELINE.json: halfspace, n=1000 Gaussian, d=5, NRandom=1000,
    # n_refinements=10, alpha=0.9, RRS seed 1, all points as queries.
    X = gen_toeplitz_gaussian(ToeplitzGaussianSpec(dim=5, n=1000, seed=0))
    cfg = df.RrsConfig(total_directions=1000, refinements=10, shrink=0.9, notion="halfspace",
                       seed=1, parallel=df.ParallelConfig(workers=os.cpu_count()))
    res = df.depth_batch(list(X), df.Dataset(X), cfg)
    out["c1_x"] = X
    out["c1_depth"] = np.array([r.depth for r in res])
    out["c1_argmin"] = np.stack([r.argmin_direction for r in res])
    out["c1_trace"] = np.stack([[np.concatenate(([t.best_depth, t.epsilon], t.pole)) for t in r.trace]
                                for r in res[:16]])

    # small cases for every notion, with traces (pole chain)
    for notion in ("halfspace", "projection", "asym_projection"):
        X = gen_toeplitz_gaussian(ToeplitzGaussianSpec(dim=4, n=257, seed=9))
        Zq = np.concatenate([X[:12], 0.5 * X[12:16], [np.zeros(4), np.full(4, 3.0)]])
        cfg = df.RrsConfig(total_directions=400, refinements=8, shrink=0.8, notion=notion, seed=77,
                           parallel=df.ParallelConfig(workers=os.cpu_count()))
        res = df.depth_batch(list(Zq), df.Dataset(X), cfg)
        out[f"rrs_{notion}_x"], out[f"rrs_{notion}_z"] = X, Zq
        out[f"rrs_{notion}_depth"] = np.array([r.depth for r in res])
        out[f"rrs_{notion}_argmin"] = np.stack([r.argmin_direction for r in res])
        out[f"rrs_{notion}_trace"] = np.stack(
            [[np.concatenate(([t.best_depth, t.epsilon], t.pole)) for t in r.trace] for r in res])

    # config 4 shape in miniature: in-sample queries are hull vertices (depth 1/n)
    X = gen_toeplitz_gaussian(ToeplitzGaussianSpec(dim=50, n=2000, seed=0))
    Zq = np.concatenate([X[:6], 0.3 * X[6:9], np.zeros((1, 50))])
    cfg = df.RrsConfig(total_directions=2000, refinements=20, shrink=0.9, notion="halfspace",
                       seed=1, parallel=df.ParallelConfig(workers=os.cpu_count()))
    res = df.depth_batch(list(Zq), df.Dataset(X), cfg)
    out["c4mini_x"], out["c4mini_z"] = X.astype(np.float64), Zq
    out["c4mini_depth"] = np.array([r.depth for r in res])

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(out)} arrays")


if __name__ == "__main__":
    main()
