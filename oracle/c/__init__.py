"""ctypes binding of the C/OpenMP oracle restatement (mo_oracle.c).  TEST INFRASTRUCTURE / CPU BASELINE
ONLY: imported by tests/ and bench.py's cpu_baseline, never by the product package."""
import ctypes
import os

import numpy as np

from . import build as _build

_L = None


def lib():
    global _L
    if _L is None:
        path = _build.LIB
        if not os.path.exists(path):
            path = _build.build()
        L = ctypes.CDLL(path)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.oro_nds.argtypes = [vp, i64, i32, i64, vp, i32]
        L.oro_dominator_counts.argtypes = [vp, i64, i32, vp, i64, vp, i32]
        L.oro_associate.argtypes = [vp, i64, i32, vp, i64, vp, vp, i64, vp, vp, i32]
        L.oro_nds3.argtypes = [vp, i64, i32, i64, vp]
        for f in (L.oro_nds, L.oro_dominator_counts, L.oro_associate, L.oro_max_threads, L.oro_nds3):
            f.restype = i32
        _L = L
    return _L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: status {rc}")


def max_threads():
    return int(lib().oro_max_threads())


def nds(F, stop_at=None, threads=0):
    """ranks (int64; 2^31-1 = dropped) like oracle.manyobj_ref.dominance.non_dominated_sort."""
    F = np.ascontiguousarray(F, np.float32)
    R, m = F.shape
    ranks = np.empty(R, np.int64)
    _check(lib().oro_nds(_p(F), R, m, int(stop_at or 0), _p(ranks), int(threads)), "oro_nds")
    return ranks


def nds3(F, stop_at=None):
    """Same ranks as :func:`nds` for m <= 3 by the lexicographic staircase sweep (mo_oracle_nds3.cc),
    O(R log R log F): the checker at C4 sizes (R = 2M), where the all-pairs sweep is minutes."""
    F = np.ascontiguousarray(F, np.float32)
    R, m = F.shape
    ranks = np.empty(R, np.int64)
    _check(lib().oro_nds3(_p(F), R, m, int(stop_at or 0), _p(ranks)), "oro_nds3")
    return ranks


def nds_auto(F, stop_at=None, threads=0):
    """nds3 for m <= 3, the all-pairs C sweep otherwise."""
    return nds3(F, stop_at) if F.shape[1] <= 3 else nds(F, stop_at, threads)


def dominator_counts(F, rows=None, threads=0):
    F = np.ascontiguousarray(F, np.float32)
    R, m = F.shape
    rr = None if rows is None else np.ascontiguousarray(rows, np.int64)
    n = R if rr is None else rr.size
    cnt = np.empty(n, np.int32)
    _check(lib().oro_dominator_counts(_p(F), R, m, None if rr is None else _p(rr), n, _p(cnt), int(threads)),
           "oro_dominator_counts")
    return cnt


def associate(Fn, zhat, pos_ref, rows=None, threads=0):
    """(pi, d) for ``rows`` (all when None) like niche.associate_canonical."""
    Fn = np.ascontiguousarray(Fn, np.float32)
    Z = np.ascontiguousarray(zhat, np.float32)
    pr = np.ascontiguousarray(pos_ref, np.int64)
    R, m = Fn.shape
    rr = None if rows is None else np.ascontiguousarray(rows, np.int64)
    n = R if rr is None else rr.size
    pi = np.empty(n, np.int64)
    d = np.empty(n, np.float32)
    _check(lib().oro_associate(_p(Fn), R, m, _p(Z), Z.shape[0], _p(pr), None if rr is None else _p(rr), n, _p(pi),
                               _p(d), int(threads)), "oro_associate")
    return pi, d


def associate_full(Fn, zhat, pos_ref, rows, threads=0):
    """Drop-in for oracle.manyobj_ref.niche.associate_canonical: full-length (pi, d) with the
    sentinels (-1, NaN) on rows not listed."""
    R = np.asarray(Fn).shape[0]
    pi = np.full(R, -1, np.int64)
    d = np.full(R, np.nan, np.float32)
    rows = np.asarray(rows, np.int64)
    if rows.size:
        p, dd = associate(Fn, zhat, pos_ref, rows=rows, threads=threads)
        pi[rows] = p
        d[rows] = dd
    return pi, d


def accel(threads=0):
    """Keyword arguments for oracle.manyobj_ref.engine.step / survivor_selection that run the
    quadratic stages here (bit-identical to the numpy restatement: tests/test_oracle_c.py,
    tests/test_oracle_fast.py)."""
    return dict(nds_fn=lambda F, stop_at: nds_auto(F, stop_at, threads),
                associate_fn=lambda Fn, zhat, pos_ref, rows: associate_full(Fn, zhat, pos_ref, rows, threads),
                fast=True)
