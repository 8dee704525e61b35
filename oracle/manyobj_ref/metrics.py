"""metrics.igd / metrics.hv restated in float64 numpy (oracle; TEST INFRASTRUCTURE ONLY).

SPEC.md:601-609 (igd: mean over reference points of the distance to the
nearest front member, O(|ref| |front|) brute force) and SPEC.md:610-618 (hv:
points that do not dominate the reference point are discarded; exact for
m <= 3 -- here by inclusion-exclusion-free slicing: m = 2 sweep, m = 3 sum
of 2-D slabs along the last objective).
"""
import numpy as np

from paper_2504_06067_b200.errors import EmptySelectionError


def igd(front, reference):
    F = np.asarray(front, np.float64)
    Z = np.asarray(reference, np.float64)
    if F.size == 0 or Z.size == 0:
        raise EmptySelectionError("igd needs nonempty inputs")
    d2 = ((Z[:, None, :] - F[None, :, :]) ** 2).sum(-1)
    return float(np.sqrt(d2.min(axis=1)).mean())


def _hv2(P, r):
    P = P[np.argsort(P[:, 0], kind="stable")]
    hv, ymin = 0.0, r[1]
    for x, y in P:
        if y < ymin:
            hv += (r[0] - x) * (ymin - y)
            ymin = y
    return hv


def hv(front, ref_point):
    """Exact hypervolume for m <= 3."""
    F = np.asarray(front, np.float64)
    r = np.asarray(ref_point, np.float64)
    F = F[(F <= r).all(axis=1)] if F.size else F.reshape(0, r.size)
    if F.shape[0] == 0:
        return 0.0
    m = r.size
    if m == 1:
        return float(r[0] - F[:, 0].min())
    if m == 2:
        return _hv2(F, r)
    if m == 3:
        zs = np.unique(F[:, 2])
        edges = np.append(zs, r[2])
        total = 0.0
        for a, b in zip(edges[:-1], edges[1:]):
            total += _hv2(F[F[:, 2] <= a][:, :2], r[:2]) * (b - a)
        return total
    raise ValueError("exact hv only for m <= 3")


def normalized_hv(fronts):
    """SPEC.md:619-627 (Appendix E Eqs. 3-5): ref = 1.01 f^max, ideal = 0.9 f^min over all fronts,
    HV_max = prod(ref - ideal); each front's exact hv / HV_max (m <= 3); HV_max = 0 -> zeros."""
    Fs = [np.asarray(f, np.float64) for f in fronts]
    allf = np.concatenate([f for f in Fs if f.size])
    ref = 1.01 * allf.max(axis=0)
    ideal = 0.9 * allf.min(axis=0)
    hv_max = float(np.prod(ref - ideal))
    if not hv_max > 0.0:
        return [0.0] * len(Fs)
    return [hv(f, ref) / hv_max for f in Fs]
