"""Reference-point lattices -- host setup, built once per run.

Not on the per-generation path: Z is built here in FP64, turned into FP32
unit directions and uploaded once.  Order: compositions of H ascending
lexicographically, outer layer before the deduplicated inner
layer.  Counting for choose_divisions uses a closed-form
duplicate count (dynamic programme over residues) instead of enumeration.
"""
from math import comb

import numpy as np

from .errors import ParameterError


def _lattice(m, H):
    """Integer compositions of H into m parts, lexicographically ascending (vectorised)."""
    rows = np.zeros((1, 0), dtype=np.int64)
    rem = np.array([H], dtype=np.int64)
    for _ in range(m - 1):
        reps = rem + 1
        new_first = np.concatenate([np.arange(r, dtype=np.int64) for r in reps]) if len(reps) else rem
        rows = np.repeat(rows, reps, axis=0)
        rem = np.repeat(rem, reps) - new_first
        rows = np.concatenate([rows, new_first[:, None]], axis=1)
    return np.concatenate([rows, rem[:, None]], axis=1)


def das_dennis(m, H):
    """All points i/H with nonnegative integers summing to H."""
    if m < 2 or H < 1:
        raise ParameterError("das_dennis needs m >= 2 and H >= 1")
    return _lattice(m, H).astype(np.float64) / float(H)


def _inner_den(m, Hi):
    return 2 * m * Hi


def two_layer(m, H_outer, H_inner):
    """Outer lattice plus inner lattice shrunk halfway to the centroid, deduplicated."""
    if m < 2 or H_outer < 1 or H_inner < 0:
        raise ParameterError("two_layer needs m >= 2, H_outer >= 1, H_inner >= 0")
    outer = _lattice(m, H_outer)
    pts = [outer.astype(np.float64) / float(H_outer)]
    if H_inner >= 1:
        num = _lattice(m, H_inner) * m + H_inner          # p/2 + 1/(2m) = num / (2 m Hi)
        den = _inner_den(m, H_inner)
        on_outer = ((num * H_outer) % den == 0).all(axis=1)
        pts.append(num[~on_outer].astype(np.float64) / float(den))
    return np.concatenate(pts, axis=0)


def _dup_count(m, Ho, Hi):
    """# compositions b of Hi whose shrunk point lies on the Ho lattice (DP over parts)."""
    if Hi < 1:
        return 0
    den = _inner_den(m, Hi)
    ok = [b for b in range(Hi + 1) if ((b * m + Hi) * Ho) % den == 0]
    ways = np.zeros(Hi + 1, dtype=object)
    ways[0] = 1
    for _ in range(m):
        nxt = np.zeros(Hi + 1, dtype=object)
        for s in range(Hi + 1):
            if ways[s]:
                for b in ok:
                    if s + b <= Hi:
                        nxt[s + b] += ways[s]
        ways = nxt
    return int(ways[Hi])


def lattice_size(m, H_outer, H_inner=0):
    n = comb(H_outer + m - 1, m - 1)
    if H_inner >= 1:
        n += comb(H_inner + m - 1, m - 1) - _dup_count(m, H_outer, H_inner)
    return n


def choose_divisions(m, n_target):
    """(H_outer, H_inner) with the largest count <= n_target.

    m <= 5: single layer (H_inner = 0).  m > 5: best two-layer pair with
    H_outer >= H_inner; ties -> larger H_outer, then larger H_inner.
    """
    if m < 2 or n_target < m:
        raise ParameterError("choose_divisions needs m >= 2 and n_target >= m")
    if m <= 5:
        H = 1
        while comb(H + m, m - 1) <= n_target:
            H += 1
        return (H, 0)
    best = None
    Ho = 1
    while comb(Ho + m - 1, m - 1) <= n_target:
        for Hi in range(Ho + 1):
            c = lattice_size(m, Ho, Hi)
            if c <= n_target and (best is None or (c, Ho, Hi) > best):
                best = (c, Ho, Hi)
        Ho += 1
    return (best[1], best[2])


def reference_points(m, n_target):
    Ho, Hi = choose_divisions(m, n_target)
    return two_layer(m, Ho, Hi) if Hi else das_dennis(m, Ho)


def unit_directions(Z):
    """zhat = z / ||z|| (FP64, fixed left-to-right sum of squares) rounded to FP32."""
    Z = np.asarray(Z, dtype=np.float64)
    if Z.ndim != 2:
        raise ParameterError("Z must be w x m")
    s = Z[:, 0] * Z[:, 0]
    for k in range(1, Z.shape[1]):
        s = s + Z[:, k] * Z[:, k]
    if (s == 0).any():
        raise ParameterError("zero reference point")
    return (Z / np.sqrt(s)[:, None]).astype(np.float32)


__all__ = ["das_dennis", "two_layer", "choose_divisions", "reference_points", "unit_directions",
           "lattice_size"]
