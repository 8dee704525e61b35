"""DTLZ1-7 batch evaluation in float64 (oracle; TEST INFRASTRUCTURE ONLY).

SPEC.md:501-528 defines DTLZ2/3/5/7; DTLZ1/4/6 follow the standard suite
(cited via PAPER.md:257).  k = d - m + 1 distance
variables (the last k), products over empty ranges are 1.
"""
from dataclasses import dataclass

import numpy as np

from paper_2504_06067_b200.errors import DomainError, ParameterError, ShapeError

KINDS = ("DTLZ1", "DTLZ2", "DTLZ3", "DTLZ4", "DTLZ5", "DTLZ6", "DTLZ7")


@dataclass(frozen=True)
class ContinuousProblem:
    """SPEC.md:506-509 (kind, m, d); bounds are [0,1]^d."""
    kind: str
    m: int
    d: int

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ParameterError(f"unknown problem {self.kind}")
        if self.d < self.m:
            raise ParameterError("d must be >= m")


def _seqsum(terms):
    """Left-to-right sum over columns (the GPU's order; numpy .sum is pairwise)."""
    s = np.zeros(terms.shape[0])
    for c in range(terms.shape[1]):
        s = s + terms[:, c]
    return s


G_LANES = 8


def _gsum(terms):
    """The g sum over the distance variables in the GPU's order: G_LANES partial sums (terms l, l+8,
    l+16, ... left to right), then the fixed pairwise tree ((p0+p4)+(p2+p6)) + ((p1+p5)+(p3+p7)) that the
    xor-shuffle butterfly of an 8-lane group computes.  (Pinned with the kernels.)"""
    n, k = terms.shape
    p = [_seqsum(terms[:, l::G_LANES]) if l < k else np.zeros(n) for l in range(G_LANES)]
    a = [p[l] + p[l + 4] for l in range(4)]
    b = [a[0] + a[2], a[1] + a[3]]
    return b[0] + b[1]


def _g_rastrigin(xm):
    k = xm.shape[1]
    t = xm - 0.5
    return 100.0 * (k + _gsum(t * t - np.cos(20.0 * np.pi * t)))


def _g_sphere(xm):
    t = xm - 0.5
    return _gsum(t * t)


def _spherical(theta, g):
    """f_j = (1+g) prod_{i<m-j} cos(theta_i) * sin(theta_{m-j}) (theta: n x (m-1))."""
    n, mm1 = theta.shape
    m = mm1 + 1
    f = np.empty((n, m))
    c = np.cos(theta)
    s = np.sin(theta)
    for j in range(m):            # j = 0 .. m-1  (objective j+1)
        v = 1.0 + g
        for i in range(m - 1 - j):
            v = v * c[:, i]
        if j > 0:
            v = v * s[:, m - 1 - j]
        f[:, j] = v
    return f


def dtlz_eval(problem, X):
    """Objective matrix n x m (float64) of DTLZ<kind> at X."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != problem.d:
        raise ShapeError("X must be n x d")
    if (X < 0).any() or (X > 1).any() or not np.isfinite(X).all():
        raise DomainError("x outside [0,1]^d")
    m = problem.m
    xp, xm = X[:, : m - 1], X[:, m - 1:]
    kind = problem.kind
    n = X.shape[0]
    if kind == "DTLZ1":
        g = _g_rastrigin(xm)
        f = np.empty((n, m))
        for j in range(m):
            v = 0.5 * (1.0 + g)
            for i in range(m - 1 - j):
                v = v * xp[:, i]
            if j > 0:
                v = v * (1.0 - xp[:, m - 1 - j])
            f[:, j] = v
        return f
    if kind in ("DTLZ2", "DTLZ3", "DTLZ4"):
        g = _g_rastrigin(xm) if kind == "DTLZ3" else _g_sphere(xm)
        pos = xp ** 100.0 if kind == "DTLZ4" else xp
        return _spherical(pos * (np.pi / 2.0), g)
    if kind in ("DTLZ5", "DTLZ6"):
        g = _g_sphere(xm) if kind == "DTLZ5" else _gsum(xm ** 0.1)
        theta = np.empty_like(xp)
        if m > 1:
            theta[:, 0] = xp[:, 0] * (np.pi / 2.0)
        for i in range(1, m - 1):
            theta[:, i] = np.pi / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xp[:, i])
        return _spherical(theta, g)
    # DTLZ7
    k = xm.shape[1]
    g = 1.0 + 9.0 / k * _gsum(xm)
    f = np.empty((n, m))
    f[:, : m - 1] = xp
    h = m - _seqsum(xp / (1.0 + g)[:, None] * (1.0 + np.sin(3.0 * np.pi * xp)))
    f[:, m - 1] = (1.0 + g) * h
    return f
