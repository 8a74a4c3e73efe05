"""depthforge-compatible RRS entry points on the B200 engine.

Same signatures, argument meaning, results and error behaviour as the
reference (optimizer.py / directions.py, cited per function); the work runs in
librrs_b200.so (sm_100a), with no CPU fallback.
"""

from __future__ import annotations

import numpy as np

from contextlib import contextmanager

from . import _lib
from .config import (CapSpec, Dataset, DepthResult, DimensionMismatch, DirectionBatch,
                     ParallelConfig, PhaseTimer, RefinementRecord, RrsConfig, NOTIONS)


@contextmanager
def _session(data: Dataset | None, device=None):
    """The device engine with `data` resident, locked for the whole call: two
    threads with different datasets must not swap the engine's dataset (or its
    workspace) between set_dataset and the compute call."""
    eng = _lib.engine(device)
    with eng.lock:
        if data is not None and eng.dataset_key is not data._token:
            eng.set_dataset(data.x, key=data._token)
        yield eng


def _results(depth, argmin, tr, cfg: RrsConfig) -> list[DepthResult]:
    m = cfg.directions_per_refinement
    out = []
    for i in range(depth.shape[0]):
        trace = tuple(RefinementRecord(best_depth=float(rec[0]), epsilon=float(rec[1]),
                                       pole=np.array(rec[2:])) for rec in tr[i])
        out.append(DepthResult(depth=float(depth[i]), argmin_direction=np.array(argmin[i]),
                               trace=trace, directions_used=m * cfg.refinements))
    return out


def _add_timer(timer: PhaseTimer | None, eng: _lib.Engine):
    if timer is None:
        return
    s = eng.stats()
    timer.add("generation", s["ms_generate"] / 1e3)
    timer.add("projection", s["ms_contract"] / 1e3)
    timer.add("univariate", (s["ms_univariate"] + s["ms_update"]) / 1e3)


def depth_batch_arrays(queries, data: Dataset, cfg: RrsConfig, *, q0: int = 0, trace: bool = False,
                       device=None, timer: PhaseTimer | None = None):
    """Array fast path of depth_batch: (depth[Q], argmin[Q,d], trace[Q,r,2+d]|None,
    min_count[Q]).  Query i uses substream q0 + i."""
    Z = np.ascontiguousarray(queries, dtype=np.float64)
    if Z.ndim == 1:
        Z = Z.reshape(1, -1)
    if Z.shape[1] != data.dim:
        raise DimensionMismatch(f"query dimension {Z.shape[1]} does not match data dimension {data.dim}")
    with _session(data, device) as eng:
        if timer is not None:
            eng.enable_timing(True)
        try:
            res = eng.depth_batch(Z, cfg, q0=q0, trace=trace, eps=cfg.epsilons())
        finally:
            if timer is not None:
                _add_timer(timer, eng)
                eng.enable_timing(False)
    return res


def depth_batch(queries, data: Dataset, cfg: RrsConfig) -> list[DepthResult]:
    """optimizer.py:254-279: element i is refined_random_search(queries[i], ...,
    query_index=i).  All queries run as device batches."""
    qs = [np.ascontiguousarray(q, dtype=np.float64).reshape(-1) for q in queries]
    for i, q in enumerate(qs):
        if q.size != data.dim:
            raise DimensionMismatch(f"query {i} has dimension {q.size}, expected {data.dim}")
    if not qs:
        return []
    depth, argmin, tr, _ = depth_batch_arrays(np.stack(qs), data, cfg, trace=True)
    return _results(depth, argmin, tr, cfg)


def refined_random_search(z, data: Dataset, cfg: RrsConfig, *, query_index: int = 0,
                          timer: PhaseTimer | None = None,
                          naive_projection: bool = False) -> DepthResult:
    """optimizer.py:145-226 (naive_projection selects the reference's
    single-thread projection; the device has one projection path)."""
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    if z.size != data.dim:
        raise DimensionMismatch(f"query dimension {z.size} does not match data dimension {data.dim}")
    depth, argmin, tr, _ = depth_batch_arrays(z[None, :], data, cfg, q0=query_index, trace=True,
                                              timer=timer)
    return _results(depth, argmin, tr, cfg)[0]


def simple_random_search(z, data: Dataset, k: int, notion: str, seed: int,
                         parallel: ParallelConfig | None = None) -> DepthResult:
    """optimizer.py:229-240: refined search with r = 1."""
    cfg = RrsConfig(total_directions=k, refinements=1, shrink=0.5, notion=notion, seed=seed,
                    parallel=parallel if parallel is not None else ParallelConfig())
    return refined_random_search(z, data, cfg)


def pole_update_rule(current, candidate):
    """optimizer.py:243-251: strict improvement; equal depth keeps the incumbent."""
    d_min, pole = current
    d_new, u_new = candidate
    if d_new < d_min:
        return d_new, u_new
    return d_min, pole


def evaluate_directions(z, data: Dataset, dirs, notion: str, cfg: ParallelConfig, *,
                        naive: bool = False, timer: PhaseTimer | None = None,
                        _buffers=None) -> np.ndarray:
    """optimizer.py:98-142: univariate depths of z over injected directions."""
    u = getattr(dirs, "directions", dirs)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.ndim != 2:
        raise DimensionMismatch("directions must form a 2-D matrix")
    if u.shape[1] != data.dim:
        raise DimensionMismatch(f"direction dimension {u.shape[1]} does not match data dimension {data.dim}")
    if notion not in NOTIONS:
        raise ValueError(f"unknown depth notion {notion!r}")
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    if z.size != data.dim:
        raise DimensionMismatch(f"query dimension {z.size} does not match data dimension {data.dim}")
    with _session(data) as eng:
        out, _, _ = eng.evaluate_directions(z, u, notion)
    if _buffers is not None:
        _buffers[2][: out.size] = out
        return _buffers[2]
    return out


def evaluate_directions_counts(z, data: Dataset, U):
    """Halfspace counts (#<=, #>=) per direction on injected directions (tier-1
    parity interface; the reference equivalent is rint(depth * n) plus
    project_parallel/project_point, projection.py:140-168)."""
    with _session(data) as eng:
        return eng.evaluate_directions(z, U, "halfspace")


def generate_batch(cap: CapSpec, m: int, seed: int, refinement: int, query: int = 0) -> DirectionBatch:
    """directions.py:192-204, generated on device (FP64)."""
    if m < 1:
        raise ValueError("batch size must be >= 1")
    with _session(None) as eng:
        U = eng.cap_directions(cap.pole.p, cap.epsilon, m, seed, refinement, query)
    return DirectionBatch(directions=U, seed_info=(seed, refinement))
