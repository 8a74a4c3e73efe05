"""Study harness and perfmodel on the host, against
the reference's own outputs (tests/golden/study_golden.npz, made by
tests/golden/make_study_golden.py) and the reference's test cases
(pkg/tests/test_correlation.py, test_perfmodel.py, test_studies.py)."""

import json
import math
import os
from itertools import combinations

import numpy as np
import pytest

import paper_2506_08262_b200 as rrs
from paper_2506_08262_b200 import perfmodel as pm
from paper_2506_08262_b200 import study

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "study_golden.npz"))


def _json(key):
    return json.loads(str(GOLD[key]))


def _tau_pairs(a, b):
    """tau-b by enumerating pairs (test oracle)."""
    con = dis = ta = tb = 0
    for i, j in combinations(range(len(a)), 2):
        da, db = np.sign(a[i] - a[j]), np.sign(b[i] - b[j])
        ta += da == 0
        tb += db == 0
        con += da * db > 0
        dis += da * db < 0
    n0 = len(a) * (len(a) - 1) // 2
    return (con - dis) / math.sqrt((n0 - ta) * (n0 - tb))


class TestCorrelation:
    def test_golden(self):
        for a, b, rho, tau in zip(GOLD["corr_a"], GOLD["corr_b"], GOLD["corr_rho"], GOLD["corr_tau"]):
            a, b = a[~np.isnan(a)], b[~np.isnan(b)]
            assert study.spearman_rho(a, b) == pytest.approx(rho, rel=1e-12, abs=1e-15)
            assert study.kendall_tau(a, b) == pytest.approx(tau, rel=1e-12, abs=1e-15)

    def test_pair_oracle_with_ties(self):
        rng = np.random.default_rng(0)
        for _ in range(60):
            n = int(rng.integers(2, 40))
            a, b = rng.integers(0, 5, n).astype(float), rng.integers(0, 5, n).astype(float)
            if np.unique(a).size < 2 or np.unique(b).size < 2:
                with pytest.raises(ValueError):
                    study.kendall_tau(a, b)
                continue
            assert study.kendall_tau(a, b) == pytest.approx(_tau_pairs(a, b), rel=1e-12, abs=1e-15)

    def test_hand_computed(self):
        assert study.spearman_rho([1, 2, 3, 4], [1, 3, 2, 4]) == pytest.approx(0.8)
        assert study.kendall_tau([1, 2, 3], [1, 3, 2]) == pytest.approx(1 / 3)
        assert study.spearman_rho([3.0, 1.0, 4.0], [3.0, 1.0, 4.0]) == 1.0
        assert study.kendall_tau([1.0, 2.0, 3.0, 4.0], [4.0, 3.0, 2.0, 1.0]) == -1.0

    def test_errors(self):
        with pytest.raises(ValueError, match="zero rank variance"):
            study.spearman_rho([1.0, 1.0, 1.0], [1.0, 2.0, 3.0])
        with pytest.raises(ValueError, match="all-tied"):
            study.kendall_tau([2.0, 2.0], [1.0, 2.0])
        with pytest.raises(ValueError, match="equal length"):
            study.kendall_tau([1.0, 2.0], [1.0, 2.0, 3.0])
        with pytest.raises(ValueError, match="at least two"):
            study.spearman_rho([1.0], [1.0])

    def test_average_ranks(self):
        np.testing.assert_array_equal(study.average_ranks(GOLD["ranks_in"]), GOLD["ranks_out"])
        np.testing.assert_array_equal(study.average_ranks([10.0, 30.0, 20.0, 20.0]), [1.0, 4.0, 2.5, 2.5])


class TestSynthetic:
    def test_generators_and_forms(self):
        spec = study.ToeplitzGaussianSpec(dim=4, n=50, seed=3)
        np.testing.assert_array_equal(study.generate(spec), GOLD["qf_queries"])
        np.testing.assert_allclose(study.quadratic_forms(spec, GOLD["qf_queries"]), GOLD["qf_out"], rtol=1e-13)
        np.testing.assert_array_equal(study.generate(study.ExponentialSpec(dim=3, n=20, seed=9)), GOLD["exp_sample"])
        tspec = study.StudentTSpec(dim=3, n=30, nu=2.5, seed=4)
        np.testing.assert_array_equal(study.generate(tspec), GOLD["t_sample"])
        np.testing.assert_array_equal(study.true_density_rank(tspec, GOLD["t_sample"]), GOLD["t_density_rank"])

    def test_validation(self):
        with pytest.raises(ValueError):
            study.ToeplitzGaussianSpec(dim=0, n=5)
        with pytest.raises(ValueError):
            study.StudentTSpec(dim=2, n=5, nu=0.0)
        with pytest.raises(TypeError):
            study.generate(object())

    def test_mahalanobis(self):
        est = rrs.estimate_mle(GOLD["t_sample"])
        np.testing.assert_allclose(rrs.mahalanobis_depth_batch(GOLD["t_sample"][:10], est), GOLD["maha_out"],
                                   rtol=1e-13)
        assert rrs.mahalanobis_depth(GOLD["t_sample"][0], est) == pytest.approx(GOLD["maha_out"][0], rel=1e-13)
        with pytest.raises(rrs.DimensionMismatch):
            rrs.mahalanobis_depth_batch(np.zeros((2, 4)), est)
        with pytest.raises(ValueError, match="not symmetric"):
            rrs.LocationScatter(location=np.zeros(2), scatter=np.array([[1.0, 0.5], [0.0, 1.0]]))
        with pytest.raises(ValueError, match="positive definite"):
            rrs.LocationScatter(location=np.zeros(2), scatter=np.array([[1.0, 2.0], [2.0, 1.0]]))


class TestPerfmodel:
    def test_golden_model(self):
        W = [pm.Workload(**w) for w in _json("pm_workloads")]
        C = pm.CostConstants(c_const=0.01, c_rv=2e-9, c_proj=3e-10, c_depth=5e-9)
        np.testing.assert_array_equal([pm.t_sequential(C, w) for w in W], GOLD["pm_tseq"])
        np.testing.assert_array_equal([pm.t_parallel(C, w) for w in W], GOLD["pm_tpar"])
        np.testing.assert_array_equal([pm.speedup(C, w) for w in W], GOLD["pm_speedup"])
        np.testing.assert_allclose([pm.speedup_plateau(C, 50, 8, 148, 1.7), pm.speedup_plateau(C, 7, 256, 16, 1.0)],
                                   GOLD["pm_plateau"], rtol=1e-15)

    def test_golden_fit(self):
        profs = [pm.TimingProfile(workload=pm.Workload(**p["w"]), generation=p["g"], projection=p["p"],
                                  univariate=p["u"], total=p["t"], path=p["path"]) for p in _json("pm_profiles")]
        rep = pm.fit_constants(profs)
        c = rep.constants
        np.testing.assert_allclose([c.c_const, c.c_rv, c.c_proj, c.c_depth, rep.r_squared, rep.max_rel_residual],
                                   GOLD["pm_fit"], rtol=1e-10)
        np.testing.assert_allclose(rep.residuals, GOLD["pm_fit_residuals"], rtol=1e-9, atol=1e-18)
        assert json.loads(rep.to_json())["profile_count"] == len(profs)

    def test_plug_in(self):
        # pkg/tests/test_perfmodel.py plug-in identities
        c1 = pm.CostConstants(c_const=0, c_rv=1, c_proj=1, c_depth=1)
        w = pm.Workload(n=5, d=7, k=6, r=2, depth_work=15)
        assert w.m == 3 and pm.t_sequential(c1, w) == 282.0
        w2 = pm.Workload(n=5, d=5, k=2, r=1, depth_work=1, g=4, lam=2.0, d_chunk=2)
        assert pm.t_parallel(pm.CostConstants(c_proj=1), w2) == 18.0
        assert pm.speedup(pm.CostConstants(c_proj=2.0, c_depth=3.0),
                          pm.Workload(n=9, d=1, k=4, r=2, g=1, lam=1.0, d_chunk=5)) == 1.0
        with pytest.raises(ValueError):
            pm.speedup(pm.CostConstants(), pm.Workload(n=1, d=1, k=1, r=1))
        with pytest.raises(ValueError):
            pm.speedup_plateau(pm.CostConstants(c_rv=1.0), 4, 2, 8, 1.0)

    def test_validation_and_rank(self):
        with pytest.raises(ValueError):
            pm.CostConstants(c_proj=-1.0)
        with pytest.raises(ValueError):
            pm.Workload(n=0, d=1, k=1)
        with pytest.raises(ValueError):
            pm.Workload(n=1, d=1, k=1, lam=0.0)
        w = pm.Workload(n=10, d=2, k=10, r=1)
        with pytest.raises(ValueError):
            pm.TimingProfile(workload=w, generation=1.0, projection=1.0, univariate=1.0, total=0.5)
        with pytest.raises(ValueError):
            pm.fit_constants([])
        few = [pm.TimingProfile(workload=w, generation=1, projection=1, univariate=1, total=4)] * 3
        with pytest.raises(pm.RankDeficientDesign) as e:
            pm.fit_constants(few)
        assert e.value.regressor == "profiles"
        same = [pm.TimingProfile(workload=w, generation=1, projection=1, univariate=1, total=4)] * 4
        with pytest.raises(pm.RankDeficientDesign) as e:
            pm.fit_constants(same)
        assert e.value.regressor == "generation"

    def test_fit_recovers_constants(self):
        C = pm.CostConstants(c_const=0.002, c_rv=1e-8, c_proj=2e-11, c_depth=4e-10)
        rng = np.random.default_rng(3)
        profs = []
        for _ in range(10):
            w = pm.Workload(n=int(rng.integers(1000, 100000)), d=int(rng.integers(2, 200)),
                            k=int(rng.integers(100, 20000)), r=int(rng.integers(1, 20)), g=148, lam=1.3, d_chunk=1)
            g, p, u = pm._terms(w, "parallel")
            profs.append(pm.TimingProfile(workload=w, generation=C.c_rv * g, projection=C.c_proj * p,
                                          univariate=C.c_depth * u, total=C.c_const + C.c_rv * g + C.c_proj * p
                                          + C.c_depth * u, path="parallel"))
        c = pm.fit_constants(profs).constants
        for a, b in ((c.c_const, C.c_const), (c.c_rv, C.c_rv), (c.c_proj, C.c_proj), (c.c_depth, C.c_depth)):
            assert a == pytest.approx(b, rel=1e-9)


class TestStudyBookkeeping:
    def test_grid_validation(self):
        ref = study.ReferenceSpec(k=1000, r=5, alpha=0.9, repeats=1)
        with pytest.raises(ValueError, match="strictly exceed"):
            study.StudyGrid(alphas=(0.9,), refinement_counts=(2,), direction_counts=(100, 1000), dims=(3,),
                            query_count=2, reference=ref)
        with pytest.raises(ValueError, match="empty"):
            study.StudyGrid(alphas=(), refinement_counts=(2,), direction_counts=(100,), dims=(3,),
                            query_count=2, reference=ref)
        with pytest.raises(ValueError):
            study.ReferenceSpec(k=3, r=5)
        with pytest.raises(ValueError):
            study.ReferenceSpec(k=30, r=5, alpha=1.0)

    def test_profile_rows_round_trip(self):
        w = [pm.Workload(n=100, d=5, k=200, r=2, g=2), pm.Workload(n=150, d=8, k=300, r=3, g=2)]
        profs = [pm.TimingProfile(workload=w[0], generation=0.1, projection=0.2, univariate=0.3, total=0.7,
                                  path="parallel")] * 2 + \
                [pm.TimingProfile(workload=w[1], generation=0.2, projection=0.1, univariate=0.3, total=0.8,
                                  path="parallel")]
        rows = study.profile_rows(profs)
        assert {r["phase"] for r in rows} == {"generation", "projection", "univariate"}
        assert len(rows) == 9
        back = study.profiles_from_rows(rows)
        assert len(back) == 3
        for a, b in zip(back, profs):   # depth_work comes back explicit, as in the reference
            assert (a.generation, a.projection, a.univariate, a.total, a.path) == \
                (b.generation, b.projection, b.univariate, b.total, b.path)
            assert a.workload.depth_units == b.workload.depth_units and a.workload.m == b.workload.m
        with pytest.raises(ValueError, match="missing phase"):
            study.profiles_from_rows(rows[:2])
        with pytest.raises(ValueError):
            study.breakdown_bench(w, "projection", "bogus")
