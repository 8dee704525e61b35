"""Reference-point lattices (oracle; TEST INFRASTRUCTURE ONLY).  SPEC.md:99-159.

Point order (pinned, shared with the product): compositions (i_1..i_m) of H in
ascending lexicographic order — matches SPEC.md:118's listing for (m=2, H=4).
Two-layer sets list the outer lattice first, then the shrunk inner lattice
with exact duplicates of outer points removed.
"""
import itertools
from math import comb, gcd

import numpy as np

from paper_2504_06067_b200.errors import ParameterError


def _compositions(m, H):
    """All m-part compositions of H, ascending lexicographic (stars and bars)."""
    out = []
    for bars in itertools.combinations(range(H + m - 1), m - 1):
        prev = -1
        row = []
        for b in bars:
            row.append(b - prev - 1)
            prev = b
        row.append(H + m - 1 - prev - 1)
        out.append(row)
    return np.array(out, dtype=np.int64).reshape(-1, m)


def das_dennis(m, H):
    """Simplex lattice {i/H : sum i = H}."""
    if m < 2 or H < 1:
        raise ParameterError("das_dennis needs m >= 2 and H >= 1")
    return _compositions(m, H).astype(np.float64) / float(H)


def _inner_numerators(m, Hi):
    """Inner point p/2 + 1/(2m) == (b*m + Hi) / (2*m*Hi) for b a composition of Hi."""
    return _compositions(m, Hi) * m + Hi


def two_layer(m, H_outer, H_inner):
    """Outer lattice U shrunk inner lattice, exact duplicates removed."""
    if m < 2 or H_outer < 1 or H_inner < 0:
        raise ParameterError("two_layer needs m >= 2, H_outer >= 1, H_inner >= 0")
    outer_int = _compositions(m, H_outer)
    pts = [outer_int.astype(np.float64) / float(H_outer)]
    if H_inner >= 1:
        num = _inner_numerators(m, H_inner)
        den = 2 * m * H_inner
        # exact duplicate test in integers: num/den == a/H_outer  <=>  num*H_outer == a*den
        outer_keys = {tuple(r) for r in (outer_int * den).tolist()}
        keep = np.array([tuple(r) not in outer_keys for r in (num * H_outer).tolist()], bool)
        pts.append(num[keep].astype(np.float64) / float(den))
    return np.concatenate(pts, axis=0)


def _dup_count(m, Ho, Hi):
    """# inner points of (Ho, Hi) lying on the outer lattice, by brute force."""
    if Hi < 1:
        return 0
    num = _inner_numerators(m, Hi)
    den = 2 * m * Hi
    return int(((num * Ho) % den == 0).all(axis=1).sum())


def two_layer_count(m, Ho, Hi):
    n = comb(Ho + m - 1, m - 1)
    if Hi >= 1:
        n += comb(Hi + m - 1, m - 1) - _dup_count(m, Ho, Hi)
    return n


def choose_divisions(m, n_target):
    """(H_outer, H_inner): largest single layer for m<=5, else best two-layer pair.

    SPEC.md:130-138.  Ties (A-11): larger w, then larger H_outer, then larger H_inner.
    """
    if m < 2 or n_target < m:
        raise ParameterError("choose_divisions needs m >= 2 and n_target >= m")
    if m <= 5:
        H = 1
        while comb(H + 1 + m - 1, m - 1) <= n_target:
            H += 1
        return (H, 0)
    best = None
    Ho = 1
    while comb(Ho + m - 1, m - 1) <= n_target:
        for Hi in range(0, Ho + 1):
            c = two_layer_count(m, Ho, Hi)
            if c <= n_target:
                key = (c, Ho, Hi)
                if best is None or key > best:
                    best = key
        Ho += 1
    return (best[1], best[2])


def reference_points(m, n_target):
    """Z for a population of n_target (single layer when H_inner == 0)."""
    Ho, Hi = choose_divisions(m, n_target)
    return two_layer(m, Ho, Hi) if Hi else das_dennis(m, Ho)


def unit_directions(Z):
    """zhat = z / ||z|| with a fixed left-to-right sum of squares, cast to FP32."""
    Z = np.asarray(Z, dtype=np.float64)
    s = Z[:, 0] * Z[:, 0]
    for k in range(1, Z.shape[1]):
        s = s + Z[:, k] * Z[:, k]
    return (Z / np.sqrt(s)[:, None]).astype(np.float32)
