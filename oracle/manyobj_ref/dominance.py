"""Pareto dominance + batched non-dominated sorting (oracle; TEST INFRASTRUCTURE ONLY).

SPEC.md:161-236.  Minimisation; duplicates are mutually non-dominating; no
epsilon.  Ranks are int64 here; DROPPED marks invalid rows and
rows in fronts beyond the split front.
"""
from dataclasses import dataclass

import numpy as np

from paper_2504_06067_b200.errors import InfeasibleSplitError, ShapeError

DROPPED = 2 ** 31 - 1


def dominates(a, b):
    """a <= b everywhere and a < b somewhere."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise ShapeError("objective vectors differ in length")
    return bool((a <= b).all() and (a < b).any())


def dominance_matrix(F, block=256):
    """M[i][j] = dominates(F[i], F[j]) as a dense bool matrix."""
    F = np.asarray(F)
    R = F.shape[0]
    M = np.zeros((R, R), dtype=bool)
    for i0 in range(0, R, block):
        A = F[i0:i0 + block, None, :]
        M[i0:i0 + block] = (A <= F[None, :, :]).all(-1) & (A < F[None, :, :]).any(-1)
    return M


def non_dominated_sort(F, valid=None, stop_at=None, block=256):
    """Iterative peeling.

    Front k = valid, unranked rows with no unranked valid dominator.  With
    ``stop_at`` (the engine's n) peeling stops at the first front whose
    cumulative size reaches it and every later row is DROPPED.
    """
    F = np.asarray(F)
    R = F.shape[0]
    valid = np.ones(R, bool) if valid is None else np.asarray(valid, bool)
    ranks = np.full(R, DROPPED, dtype=np.int64)
    vidx = np.flatnonzero(valid)
    Fv = F[vidx]
    D = np.zeros((len(vidx), len(vidx)), dtype=bool)
    for i0 in range(0, len(vidx), block):
        A = Fv[i0:i0 + block, None, :]
        D[i0:i0 + block] = (A <= Fv[None, :, :]).all(-1) & (A < Fv[None, :, :]).any(-1)
    cnt_v = D.sum(axis=0).astype(np.int64)
    unranked = np.ones(len(vidx), bool)
    cum = 0
    k = 0
    while unranked.any():
        front = unranked & (cnt_v == 0)
        ranks[vidx[front]] = k
        unranked &= ~front
        cum += int(front.sum())
        cnt_v -= D[front].sum(axis=0)
        if stop_at is not None and cum >= stop_at:
            break
        k += 1
    return ranks


@dataclass(frozen=True)
class FrontSplit:
    """SPEC.md:172-175 (l, selected_count, k)."""
    l: int
    selected_count: int
    k: int


def split_fronts(ranks, n):
    """l = first front with cumulative >= n; selected = cum(<l); k = n - selected."""
    ranks = np.asarray(ranks)
    live = ranks[ranks != DROPPED]
    if live.size < n:
        raise InfeasibleSplitError(f"{live.size} valid individuals < n={n}")
    sizes = np.bincount(live, minlength=int(live.max()) + 1 if live.size else 0)
    cum = np.cumsum(sizes)
    l = int(np.searchsorted(cum, n))        # first index with cum >= n
    sel = int(cum[l - 1]) if l > 0 else 0
    return FrontSplit(l, sel, n - sel)


def front_sizes(ranks):
    live = np.asarray(ranks)[np.asarray(ranks) != DROPPED]
    return np.bincount(live) if live.size else np.zeros(0, np.int64)
