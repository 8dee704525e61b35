"""NSGA-III niching on the GPU: Alg. 2.

The engine runs these stages fused inside ``mo_step``; the functions here
expose them one by one with the reference's op names for parity testing and
for callers that hold their own ranks.  All index tie-breaks use the keyed
shuffles of (seed, generation).

``oracle_niche_select`` (Alg. 1) is deliberately absent:
it is the CPU test oracle (oracle/manyobj_ref/niche.py), not an engine path.
"""
import torch

from . import _lib
from ._tensor import as_cuda, as_matrix
from .dominance import DROPPED
from .errors import ParameterError, ShapeError


def _ranks_info(R, ranks, l, device):
    if ranks is None:
        ranks = torch.zeros(R, dtype=torch.int32, device=device)
        l = 0
    else:
        ranks = as_cuda(ranks, torch.int32)
        if ranks.shape != (R,):
            raise ShapeError("ranks must have one entry per row")
        if l is None:
            raise ParameterError("l is required with ranks")
    return ranks, _lib.new_info(device, L=l)


def normalize_objectives(F, ideal=None, ranks=None, l=None, seed=0, generation=0):
    """(Fn, ideal, intercepts) over candidate rows (rank <= l; all rows if ranks is None).

    SPEC.md:331-339 with DESIGN.md's pins: FP32 running-min ideal over all
    rows, ASF extremes (ties -> lowest shuffled position), FP64 hyperplane
    solve, per-component fallbacks.  Non-candidate rows of Fn are NaN.
    """
    F = as_matrix(F)
    R, m = F.shape
    dev = F.device
    ideal = (torch.full((m,), float("inf"), dtype=torch.float32, device=dev) if ideal is None
             else as_cuda(ideal, torch.float32).clone())
    ranks, info = _ranks_info(R, ranks, l, dev)
    Fn = torch.full((R, m), float("nan"), dtype=torch.float32, device=dev)
    icpt = torch.empty(m, dtype=torch.float64, device=dev)
    ws = _lib.workspace_rows(R, m, 1, dev)
    _lib.check(_lib.lib().mo_normalize(_lib.ptr(F), R, m, _lib.ptr(ranks), _lib.ptr(info), int(seed),
                                       int(generation), _lib.ptr(ideal), _lib.ptr(Fn), _lib.ptr(icpt),
                                       _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "mo_normalize")
    return Fn, ideal, icpt


def associate(Fn, zhat, ranks=None, l=None, seed=0, generation=0):
    """(pi, d) per candidate row -- fused Eq. (2) distance + argmin.

    pi = nearest reference point by the canonical FP32 key (ties -> lowest
    shuffled reference position), d = perpendicular distance.  Rows that are
    not candidates get pi = -1, d = NaN (the sentinel of SPEC.md:357).
    """
    Fn = as_matrix(Fn)
    zhat = as_matrix(zhat)
    R, m = Fn.shape
    w = zhat.shape[0]
    if zhat.shape[1] != m:
        raise ShapeError("zhat must be w x m")
    dev = Fn.device
    ranks, info = _ranks_info(R, ranks, l, dev)
    pi = torch.full((R,), -1, dtype=torch.int32, device=dev)
    d = torch.full((R,), float("nan"), dtype=torch.float32, device=dev)
    ws = _lib.workspace_rows(R, m, w, dev)
    _lib.check(_lib.lib().mo_associate(_lib.ptr(Fn), R, m, _lib.ptr(zhat), w, _lib.ptr(ranks), _lib.ptr(info),
                                       int(seed), int(generation), _lib.ptr(pi), _lib.ptr(d), _lib.ptr(ws),
                                       ws.numel(), _lib.stream_ptr()), "mo_associate")
    return pi, d


def niche_select(pi, d, ranks, split, n, w, seed=0, generation=0):
    """niche_counts + nearest_selection + build_cache + batched_random_selection.

    ``split`` is the FrontSplit of ``ranks``.  Returns (selected bool mask,
    updated ranks with promoted rows at l-1, info dict).
    """
    pi = as_cuda(pi, torch.int32)
    d = as_cuda(d, torch.float32)
    ranks = as_cuda(ranks, torch.int32).clone()
    R = ranks.shape[0]
    dev = ranks.device
    fl = int((ranks == split.l).sum().item())
    info = _lib.new_info(dev, L=split.l, SELECTED=split.selected_count, K=split.k, FL_SIZE=fl,
                         SKIPPED=int(split.selected_count + fl == n))
    sel = torch.zeros(R, dtype=torch.uint8, device=dev)
    ws = _lib.workspace_rows(R, 1, w, dev)
    _lib.check(_lib.lib().mo_niche_select(_lib.ptr(pi), _lib.ptr(d), R, int(w), int(n), _lib.ptr(ranks),
                                          _lib.ptr(info), int(seed), int(generation), _lib.ptr(sel), _lib.ptr(ws),
                                          ws.numel(), _lib.stream_ptr()), "mo_niche_select")
    h = info.cpu().tolist()
    return sel.bool(), ranks, {k: h[v] for k, v in _lib.INFO.items()}


def perpendicular_distance_matrix(Fn, Z):
    """Materialised D[i][j] = ||f|| sqrt(1 - cos^2), for small inputs / API parity.

    Evaluated as the rejection length ||f - (f . zhat) zhat|| (no 1 - cos^2
    cancellation).  The engine never builds D (it would be 8 TB at N=1M); it
    uses the fused association of :func:`associate`.
    """
    Fn = as_matrix(Fn, torch.float64)
    Z = as_matrix(Z, torch.float64)
    zn = Z.norm(dim=1)
    if (zn == 0).any():
        raise ParameterError("zero reference point")
    zh = Z / zn[:, None]
    t = Fn @ zh.t()
    E = Fn[:, None, :] - t[:, :, None] * zh[None, :, :]
    return E.norm(dim=2)


__all__ = ["normalize_objectives", "associate", "niche_select", "perpendicular_distance_matrix", "DROPPED"]
