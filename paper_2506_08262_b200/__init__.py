"""B200-native Refined Random Search (RRS) for projection-based depths
(arXiv 2506.08262), a drop-in for depthforge's RRS hot path.

depthforge-compatible names (optimizer.py / projection.py / directions.py):
    RrsConfig, ParallelConfig, Dataset, DimensionMismatch, DepthResult,
    RefinementRecord, PhaseTimer, depth_batch, refined_random_search,
    evaluate_directions, simple_random_search, pole_update_rule,
    generate_batch, Pole, CapSpec, DirectionBatch, SubStream, random_sphere,
    random_sphere_pole (directions.py); ProjectionMatrix, project_naive,
    project_parallel, project_point (projection.py; module projection_ops);
    ProjectedSample, depth_of_projections,
    halfspace/projection/asym_projection_depth_1d
    (univariate.py)
    perfmodel (perfmodel.py): CostConstants, Workload, TimingProfile, t_sequential,
    t_parallel, speedup, speedup_plateau, fit_constants, FitReport
    Mahalanobis baseline (univariate.py): LocationScatter, estimate_mle,
    mahalanobis_depth, mahalanobis_depth_batch
    study harness (study/): rank_study, convergence_study, convergence_frontier,
    breakdown_bench, runtime_grid, spearman_rho, kendall_tau, synthetic specs
data-depth-style wrappers:
    halfspace, projection, aprojection (NRandom, n_refinements, sphcap_shrink,
    solver="refinedrandom")

All compute runs in the sm_100a C-ABI library librrs_b200.so (built in-tree,
see build.py); there is no CPU fallback.
"""

from ._lib import Engine, LibraryNotBuilt, device_count, engine, load_library
from .config import (CapSpec, Dataset, DepthResult, DimensionMismatch, DirectionBatch, NOTIONS,
                     ParallelConfig, PhaseTimer, Pole, RefinementRecord, RrsConfig)
from .datadepth import aprojection, halfspace, projection
from .directions import SubStream, random_sphere, random_sphere_pole
from .projection_ops import ProjectionMatrix, project_naive, project_parallel, project_point
from .univariate import (ProjectedSample, asym_projection_depth_1d, depth_of_projections, halfspace_depth_1d,
                         projection_depth_1d)
from .mahalanobis import LocationScatter, estimate_mle, mahalanobis_depth, mahalanobis_depth_batch
from .perfmodel import (CostConstants, FitReport, RankDeficientDesign, TimingProfile, Workload, fit_constants,
                        speedup, speedup_plateau, t_parallel, t_sequential)
from .solver import (depth_batch, depth_batch_arrays, evaluate_directions, evaluate_directions_counts,
                     generate_batch, pole_update_rule, refined_random_search, simple_random_search)


def backend_name() -> str:
    """_core/__init__.py:25 analogue: the only backend is the B200 library."""
    return "b200"


__version__ = "0.1.0"

__all__ = [
    "CostConstants", "FitReport", "LocationScatter", "RankDeficientDesign", "TimingProfile", "Workload",
    "estimate_mle", "fit_constants", "mahalanobis_depth", "mahalanobis_depth_batch", "speedup",
    "speedup_plateau", "t_parallel", "t_sequential",
    "CapSpec", "Dataset", "DepthResult", "DimensionMismatch", "DirectionBatch", "Engine",
    "LibraryNotBuilt", "NOTIONS", "ParallelConfig", "PhaseTimer", "Pole", "RefinementRecord",
    "RrsConfig", "aprojection", "backend_name", "depth_batch", "depth_batch_arrays", "device_count",
    "engine", "evaluate_directions", "evaluate_directions_counts", "generate_batch", "halfspace",
    "load_library", "pole_update_rule", "projection", "refined_random_search", "simple_random_search",
    "ProjectedSample", "ProjectionMatrix", "SubStream", "asym_projection_depth_1d", "depth_of_projections",
    "halfspace_depth_1d", "project_naive", "project_parallel", "project_point", "projection_depth_1d",
    "random_sphere", "random_sphere_pole",
]
