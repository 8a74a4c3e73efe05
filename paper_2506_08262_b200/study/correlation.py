"""Rank correlations for the rank study (reference study/correlation.py:1-105):
Spearman's rho (Pearson correlation of average ranks) and Kendall's tau-b.

tau-b = (n0 - t_a - t_b + t_ab - 2 D) / sqrt((n0 - t_a)(n0 - t_b)), n0 = n(n-1)/2,
t_a / t_b the pairs tied in a / in b, t_ab the pairs tied in both, D the
strictly discordant pairs.  D is counted here with a Fenwick tree over the
dense ranks of b, visiting the observations in (a, b) order: an earlier
observation with a strictly larger b is a discordant pair (pairs tied in a are
ordered by b, so they never count).  O(n log n) like the reference's merge
sort; same value.
"""

from __future__ import annotations

import math

import numpy as np

from .synthetic import average_ranks


def _vector(x, name: str) -> np.ndarray:
    v = np.asarray(x, dtype=np.float64).reshape(-1)
    if v.size < 2:
        raise ValueError(f"{name} needs at least two entries")
    return v


def _pair(a, b) -> tuple[np.ndarray, np.ndarray]:
    av, bv = _vector(a, "a"), _vector(b, "b")
    if av.size != bv.size:
        raise ValueError("inputs must have equal length")
    return av, bv


def spearman_rho(a, b) -> float:
    """Pearson correlation of average ranks; ValueError on zero rank variance."""
    av, bv = _pair(a, b)
    ra = average_ranks(av)
    rb = average_ranks(bv)
    ra -= ra.mean()
    rb -= rb.mean()
    va, vb = float(ra @ ra), float(rb @ rb)
    if va == 0.0 or vb == 0.0:
        raise ValueError("zero rank variance")
    return float(ra @ rb) / math.sqrt(va * vb)


def _tied_pairs(run_lengths: np.ndarray) -> int:
    c = run_lengths.astype(np.int64)
    return int((c * (c - 1) // 2).sum())


def _runs(*keys_sorted: np.ndarray) -> np.ndarray:
    """Lengths of the runs of equal (key, ...) tuples in sorted arrays."""
    n = keys_sorted[0].size
    brk = np.zeros(n - 1, dtype=bool)
    for k in keys_sorted:
        brk |= k[1:] != k[:-1]
    edges = np.concatenate(([0], np.flatnonzero(brk) + 1, [n]))
    return np.diff(edges)


def _discordant(b_in_a_order: np.ndarray) -> int:
    """#(i < j with b_i > b_j) by a Fenwick tree over dense ranks of b."""
    _, dense = np.unique(b_in_a_order, return_inverse=True)
    size = int(dense.max()) + 1
    tree = [0] * (size + 1)
    seen = 0
    inv = 0
    for r in dense.tolist():
        # count seen values with rank <= r
        i, le = r + 1, 0
        while i > 0:
            le += tree[i]
            i -= i & -i
        inv += seen - le
        i = r + 1
        while i <= size:
            tree[i] += 1
            i += i & -i
        seen += 1
    return inv


def kendall_tau(a, b) -> float:
    """Tie-corrected tau-b; ValueError when either input is all ties."""
    av, bv = _pair(a, b)
    n = av.size
    n0 = n * (n - 1) // 2
    order = np.lexsort((bv, av))
    a_s, b_s = av[order], bv[order]
    t_a = _tied_pairs(_runs(a_s))
    t_b = _tied_pairs(_runs(np.sort(bv)))
    t_ab = _tied_pairs(_runs(a_s, b_s))
    den_a, den_b = n0 - t_a, n0 - t_b
    if den_a == 0 or den_b == 0:
        raise ValueError("kendall tau undefined for an all-tied vector")
    disc = _discordant(b_s)
    return (n0 - t_a - t_b + t_ab - 2 * disc) / math.sqrt(den_a * den_b)
