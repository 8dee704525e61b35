"""Quality indicators (the reference's ``metrics`` module)
and the DTLZ Pareto-front samplers IGD needs (``problems.dtlz_pf_sample``,
SPEC.md:529-537) -- SURVEY.md 8(f) item 1.

* :func:`igd` runs on the GPU (``mo_igd``: fused min-distance reduction in
  FP64, deterministic), like the association kernel it resembles.
* :func:`hv`: exact for m <= 3 on the GPU (``mo_hv_exact``:
  slab decomposition, FP64, deterministic), Monte-Carlo with 10^6 samples and
  a fixed seed for m > 3 (:func:`hv_mc`, ``mo_hv_mc``: Philox samples,
  dominance counts; it also returns the standard error).
* :func:`normalized_hv` (the paper's Appendix E Eqs. 3-5).
* :func:`dtlz_pf_sample` is host set-up code like ``refpoints``: FP64 points
  on the true front from the problems' own parametrisations at g = 0,
  positions from the R_(m-1) Kronecker sequence (deterministic, low
  discrepancy).  DTLZ7's front is the non-dominated part of its g = 0
  surface, so candidates are filtered (in order) until ``count`` remain.
"""
import ctypes
import warnings

import numpy as np
import torch

from . import _lib
from ._tensor import as_matrix
from .errors import EmptySelectionError, ParameterError, ShapeError


def igd(front, reference):
    """Mean over ``reference`` rows of the distance to the nearest ``front`` row."""
    F = as_matrix(front)
    Z = as_matrix(reference)
    if F.shape[0] == 0 or Z.shape[0] == 0:
        raise EmptySelectionError("igd needs a nonempty front and reference")
    if F.shape[1] != Z.shape[1]:
        raise ShapeError("front and reference must have the same number of objectives")
    L = _lib.lib()
    ws = torch.empty(int(L.mo_igd_workspace_bytes(Z.shape[0])), dtype=torch.uint8, device=F.device)
    out = torch.empty(1, dtype=torch.float64, device=F.device)
    _lib.check(L.mo_igd(_lib.ptr(F), F.shape[0], _lib.ptr(Z), Z.shape[0], F.shape[1], _lib.ptr(out), _lib.ptr(ws),
                        ws.numel(), _lib.stream_ptr()), "mo_igd")
    return float(out.item())


def hv_mc(front, ref_point, samples=10 ** 6, seed=0, lower=None):
    """Monte-Carlo hypervolume (m > 3 branch): rows that do not dominate ``ref_point``
    are discarded; ``samples`` points uniform in [lower, ref_point] (lower = column minima of the
    retained rows).  Returns (hv, standard error)."""
    F = as_matrix(front)
    r = torch.as_tensor(np.asarray(ref_point, np.float64), device=F.device)
    if r.numel() != F.shape[1]:
        raise ShapeError("ref_point must have one component per objective")
    keep = (F.double() <= r).all(dim=1)
    Fk = F[keep].contiguous()
    if Fk.shape[0] == 0:
        return 0.0, 0.0
    lo = Fk.double().amin(dim=0) if lower is None else torch.as_tensor(np.asarray(lower, np.float64),
                                                                        device=F.device)
    lo = lo.contiguous()
    L = _lib.lib()
    ws = torch.empty(int(L.mo_hv_mc_workspace_bytes(int(samples))), dtype=torch.uint8, device=F.device)
    hits = torch.zeros(1, dtype=torch.int64, device=F.device)
    _lib.check(L.mo_hv_mc(_lib.ptr(Fk), Fk.shape[0], F.shape[1], _lib.ptr(lo), _lib.ptr(r), int(samples),
                          ctypes.c_uint64(int(seed)), _lib.ptr(hits), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "mo_hv_mc")
    vol = float(torch.prod(r - lo).item())
    p = int(hits.item()) / float(samples)
    return vol * p, vol * np.sqrt(max(p * (1.0 - p), 0.0) / samples)


def hv(front, ref_point, samples=10 ** 6, seed=0):
    """Hypervolume dominated by ``front`` and bounded by ``ref_point``: rows that do
    not weakly dominate ``ref_point`` are discarded (empty -> 0).  m <= 3: exact; m > 3: the
    Monte-Carlo estimate of :func:`hv_mc` (``samples``, fixed ``seed``)."""
    F = as_matrix(front)
    m = F.shape[1]
    r = np.asarray(ref_point, np.float64).reshape(-1)
    if r.size != m:
        raise ShapeError("ref_point must have one component per objective")
    if m > 3:
        return hv_mc(F, r, samples=samples, seed=seed)[0]
    if F.shape[0] == 0:
        return 0.0
    L = _lib.lib()
    rd = torch.as_tensor(r, device=F.device)
    ws = torch.empty(int(L.mo_hv_exact_workspace_bytes(F.shape[0])), dtype=torch.uint8, device=F.device)
    out = torch.empty(1, dtype=torch.float64, device=F.device)
    _lib.check(L.mo_hv_exact(_lib.ptr(F), F.shape[0], m, _lib.ptr(rd), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                             _lib.stream_ptr()), "mo_hv_exact")
    return float(out.item())


def normalized_hv(fronts, samples=10 ** 6, seed=0):
    """SPEC.md:619-627 / Appendix E Eqs. (3)-(5): f^max, f^min over ALL fronts; ref = 1.01 f^max,
    ideal = 0.9 f^min (applied literally, also to negative minima), HV_max = prod(ref - ideal); each
    front's hv(front, ref) / HV_max.  HV_max = 0 -> all zeros and a RuntimeWarning."""
    Fs = [as_matrix(f) for f in fronts]
    if not Fs:
        raise EmptySelectionError("normalized_hv needs at least one front")
    m = Fs[0].shape[1]
    if any(f.shape[1] != m for f in Fs):
        raise ShapeError("all fronts must have the same number of objectives")
    rows = [f.double() for f in Fs if f.shape[0] > 0]
    if not rows:
        raise EmptySelectionError("normalized_hv needs a nonempty front")
    allf = torch.cat(rows)
    fmax = allf.amax(dim=0).cpu().numpy()
    fmin = allf.amin(dim=0).cpu().numpy()
    ref = 1.01 * fmax
    ideal = 0.9 * fmin
    hv_max = float(np.prod(ref - ideal))
    if not hv_max > 0.0:
        warnings.warn("normalized_hv: HV_max = 0 (degenerate fronts); all values set to 0", RuntimeWarning)
        return [0.0] * len(Fs)
    return [hv(f, ref, samples=samples, seed=seed) / hv_max for f in Fs]


# ------------------------------------------------------------- front samplers

def _kronecker(count, dim):
    """R_dim sequence: frac(0.5 + n * alpha), alpha_i = phi_dim^-(i+1) (phi_dim: x^(dim+1) = x + 1)."""
    if dim == 0:
        return np.zeros((count, 0))
    phi = 2.0
    for _ in range(60):
        phi = (1.0 + phi) ** (1.0 / (dim + 1))
    alpha = phi ** -np.arange(1, dim + 1, dtype=np.float64)
    n = np.arange(1, count + 1, dtype=np.float64)[:, None]
    return np.mod(0.5 + n * alpha[None, :], 1.0)


def _spherical(x, radius=1.0):
    """DTLZ2 shape at g = 0: f_j = prod_{i<m-j} cos(x_i pi/2) * sin(x_{m-j} pi/2) (j >= 1)."""
    n, mm1 = x.shape
    m = mm1 + 1
    c, s = np.cos(x * np.pi / 2), np.sin(x * np.pi / 2)
    f = np.empty((n, m))
    for j in range(m):
        v = np.full(n, radius)
        for i in range(m - 1 - j):
            v = v * c[:, i]
        if j > 0:
            v = v * s[:, m - 1 - j]
        f[:, j] = v
    return f


def _nondominated_mask(F):
    n = F.shape[0]
    keep = np.ones(n, bool)
    for i in range(n):
        if keep[i]:
            dom = (F[i] <= F).all(1) & (F[i] < F).any(1)
            keep &= ~dom
    return keep


def dtlz_pf_sample(kind, m, count):
    """``count`` FP64 points on the Pareto front of DTLZ ``kind`` with m objectives."""
    if count < 1 or m < 2:
        raise ParameterError("dtlz_pf_sample needs count >= 1 and m >= 2")
    if kind == "DTLZ1":                                  # hyperplane sum f = 1/2
        x = _kronecker(count, m - 1)
        f = np.empty((count, m))
        for j in range(m):
            v = np.full(count, 0.5)
            for i in range(m - 1 - j):
                v = v * x[:, i]
            if j > 0:
                v = v * (1.0 - x[:, m - 1 - j])
            f[:, j] = v
        return f
    if kind in ("DTLZ2", "DTLZ3", "DTLZ4"):              # unit sphere, positive orthant
        return _spherical(_kronecker(count, m - 1))
    if kind in ("DTLZ5", "DTLZ6"):                       # degenerate curve: theta_i = pi/4 for i >= 2
        x = np.full((count, m - 1), 0.5)
        x[:, 0] = _kronecker(count, 1)[:, 0] if count > 1 else 0.5
        return _spherical(x)
    if kind == "DTLZ7":                                  # non-dominated part of the g = 1 surface
        out = []
        have = 0
        batch = max(4 * count, 64)
        start = 0
        while have < count:
            u = _kronecker(start + batch, m - 1)[start:]
            f = np.empty((u.shape[0], m))
            f[:, :m - 1] = u
            f[:, m - 1] = 2.0 * (m - np.sum(u / 2.0 * (1.0 + np.sin(3.0 * np.pi * u)), axis=1))
            out.append(f)
            allf = np.concatenate(out)
            keep = _nondominated_mask(allf)
            have = int(keep.sum())
            start += batch
        return allf[keep][:count]
    raise ParameterError(f"no closed-form front for {kind!r}")


__all__ = ["igd", "hv", "hv_mc", "normalized_hv", "dtlz_pf_sample"]
