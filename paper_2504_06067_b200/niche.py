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
from ._tensor import as_cuda, as_mask, as_matrix
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


def associate_canonical(Fn, zhat, ranks=None, l=None, seed=0, generation=0):
    """(pi, d) per candidate row -- fused Eq. (2) distance + argmin; the oracle's
    ``associate_canonical`` (oracle/manyobj_ref/niche.py:168) with the shuffles keyed by (seed,
    generation) as in the engine.

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


def associate(D, valid=None):
    """SPEC.md:349-357 over a materialised distance matrix (R x w): per valid row pi = argmin (lowest
    column on ties), d = the minimum; invalid rows get the sentinel (-1, NaN).  int64 / FP64 CUDA
    tensors.  (The engine never builds D; see :func:`associate_canonical`.)"""
    D = as_matrix(D, torch.float64)
    R, w = D.shape
    if w < 1:
        raise ShapeError("D needs at least one column")
    v = as_mask(valid, R)
    pi = torch.empty(R, dtype=torch.int64, device=D.device)
    d = torch.empty(R, dtype=torch.float64, device=D.device)
    _lib.check(_lib.lib().mo_associate_matrix(_lib.ptr(D), _lib.ptr(v), R, w, _lib.ptr(pi), _lib.ptr(d),
                                              _lib.stream_ptr()), "mo_associate_matrix")
    return pi, d


def _i64(x):
    return as_cuda(x, torch.int64)


def niche_counts(pi, ranks, l, w):
    """(rho, rho') int64 over w points; rho counts rank < l (when l > 0), rho' counts
    rank == l, and rho = INF (2^31 - 1) wherever rho' = 0."""
    pi, ranks = _i64(pi), _i64(ranks)
    if pi.shape != ranks.shape:
        raise ShapeError("pi and ranks need one entry per row")
    dev = pi.device
    rho = torch.empty(int(w), dtype=torch.int64, device=dev)
    rho_p = torch.empty(int(w), dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().mo_niche_counts(_lib.ptr(pi), _lib.ptr(ranks), pi.numel(), int(l), int(w), _lib.ptr(rho),
                                          _lib.ptr(rho_p), _lib.stream_ptr()), "mo_niche_counts")
    return rho, rho_p


def nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref):
    """SPEC.md:367-375 (Alg. 2 lines 8-12): returns (promoted rows, rho, rho') -- for every point with
    rho = 0 its rank-l candidate of smallest (d, shuffled position); all of them when they fit in
    k (point order), else the first k in shuffled reference order."""
    pi, ranks, pos_pop, pos_ref = _i64(pi), _i64(ranks), _i64(pos_pop), _i64(pos_ref)
    d = as_cuda(d, torch.float32)
    rho, rho_p = _i64(rho).clone(), _i64(rho_p).clone()
    R, w = pi.numel(), rho.numel()
    dev = pi.device
    promoted = torch.empty(w, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = _lib.workspace_ops(R, w, dev)
    _lib.check(_lib.lib().mo_nearest_selection(_lib.ptr(pi), _lib.ptr(d), _lib.ptr(ranks), R, int(l), _lib.ptr(rho),
                                               _lib.ptr(rho_p), w, int(k), _lib.ptr(pos_pop), _lib.ptr(pos_ref),
                                               _lib.ptr(promoted), _lib.ptr(cnt), _lib.ptr(ws), ws.numel(),
                                               _lib.stream_ptr()), "mo_nearest_selection")
    return promoted[: int(cnt.item())], rho, rho_p


def build_cache(pi, ranks, l, w, pos_pop, exclude=None):
    """the cache table as CSR (offsets[w+1], cand) -- rank-l rows not in ``exclude``
    (row indices), grouped by reference point, shuffled population order inside a point."""
    pi, ranks, pos_pop = _i64(pi), _i64(ranks), _i64(pos_pop)
    R = pi.numel()
    dev = pi.device
    ex = None
    if exclude is not None:
        e = _i64(exclude)
        ex = torch.zeros(R, dtype=torch.uint8, device=dev)
        if e.numel():
            ex[e] = 1
    offsets = torch.empty(int(w) + 1, dtype=torch.int64, device=dev)
    cand = torch.empty(max(R, 1), dtype=torch.int64, device=dev)
    ws = _lib.workspace_ops(R, w, dev)
    _lib.check(_lib.lib().mo_build_cache(_lib.ptr(pi), _lib.ptr(ranks), R, int(l), int(w), _lib.ptr(pos_pop),
                                         _lib.ptr(ex), _lib.ptr(offsets), _lib.ptr(cand), _lib.ptr(ws), ws.numel(),
                                         _lib.stream_ptr()), "mo_build_cache")
    return offsets, cand[: int(offsets[-1].item())]


def batched_random_selection(offsets, cand, rho, rho_p, k, pos_ref):
    """SPEC.md:385-393 (Alg. 2 lines 15-26): (taken rows in the loop's order, loop iterations).
    Raises InfeasibleSplitError when the points run out before k rows are taken."""
    offsets, cand, rho, rho_p, pos_ref = _i64(offsets), _i64(cand), _i64(rho), _i64(rho_p), _i64(pos_ref)
    w, k = rho.numel(), int(k)
    dev = rho.device
    taken = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    info = torch.zeros(3, dtype=torch.int64, device=dev)
    ws = _lib.workspace_ops(k, w, dev)
    _lib.check(_lib.lib().mo_batched_random_selection(_lib.ptr(offsets), _lib.ptr(cand), _lib.ptr(rho),
                                                      _lib.ptr(rho_p), w, k, _lib.ptr(pos_ref), _lib.ptr(taken),
                                                      _lib.ptr(info), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "mo_batched_random_selection")
    h = info.tolist()
    _lib.check(h[2], "batched_random_selection")
    return taken[: h[0]], h[1]


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


__all__ = ["normalize_objectives", "associate", "associate_canonical", "niche_counts", "nearest_selection",
           "build_cache", "batched_random_selection", "niche_select", "perpendicular_distance_matrix", "DROPPED"]


# ------------------------------------------------------------------ debug bookkeeping / niche trace

def niche_state(engine):
    """Views of the niche-selection state the engine's last step left in its workspace (valid until the
    next step): pi, d, prom (per merged row); rho, rho_p (post-nearest counts), take (cache entries taken)
    per reference point; the row / reference positions of that generation's shuffles."""
    cfg = engine.cfg
    n, m, w = cfg.n, cfg.m, engine.w
    R = 2 * n
    off = _lib.niche_offsets(n, m, w, engine.sort_mode, engine.shard_count)
    ws = engine.ws

    def i32(name, count):
        return ws[off[name]: off[name] + 4 * count].view(torch.int32)
    return {"pi": i32("pi", R), "d": ws[off["d"]: off["d"] + 4 * R].view(torch.float32),
            "prom": ws[off["prom"]: off["prom"] + R].bool(), "rho": i32("rho", w), "rho_p": i32("rho_p", w),
            "take": i32("take", w), "pos_pop": i32("pos_pop", R), "pos_ref": i32("pos_ref", w)}


def trace(engine):
    """The SPEC debug trace record of the last step's niching: post-nearest counts rho /
    rho', the per-point takes, the water level L* (the batched loop's iterations collapse into it) and
    the promoted rows.  A plain dict (host lists), one record per generation."""
    info = engine.info_dict()
    st = niche_state(engine)
    return {"generation": engine.generation - 1, "l": info["l"], "k": info["k"], "nearest": info["nearest"],
            "level": info["level"], "skipped": info["skipped"], "rho": st["rho"].tolist(),
            "rho_prime": st["rho_p"].tolist(), "take": st["take"].tolist(),
            "promoted": torch.nonzero(st["prom"]).flatten().tolist()}


def check_bookkeeping(engine):
    """SPEC.md:406's debug-mode check, in the closed form the engine computes: recompute from scratch
    (from the final ranks, the association and the promoted flags of the last step) the niche counts over
    F_s, the nearest-selection outcome, the post-nearest counts rho / rho', the per-point takes against
    the water level, the cache order (the taken members of a point are its take_j lowest shuffled
    positions) and the survivor count.  Returns {check: bool}; all True on a consistent step."""
    info = engine.info_dict()
    n, w = engine.cfg.n, engine.w
    out = {"survivors": info["survivors"] == n}
    if info["skipped"]:
        return out
    st = niche_state(engine)
    l, k = info["l"], info["k"]
    ranks = engine.ranks
    prom = st["prom"]
    orig = torch.where(prom, torch.full_like(ranks, l), ranks)
    Fs = (orig >= 0) & (orig < l)
    Fl = orig == l
    pi = st["pi"].long()
    rho0 = torch.bincount(pi[Fs], minlength=w)[:w]
    rhop0 = torch.bincount(pi[Fl], minlength=w)[:w]
    empty = (rho0 == 0) & (rhop0 > 0)
    M0 = int(empty.sum())
    out["final_ranks"] = bool((ranks < l).sum() == n)   # promoted rows carry l - 1 (-1 when l = 0)
    # nearest candidate of every empty niche: min (d, shuffled position) over its F_l members
    R = ranks.numel()
    pos = st["pos_pop"].long()
    rows = torch.nonzero(Fl).flatten()
    d = st["d"][rows].double()
    key = pi[rows] * (R + 1) + pos[rows]               # group by niche, ties by shuffled position
    order = torch.argsort(key)
    order = order[torch.sort(d[order], stable=True).indices]
    grp = pi[rows][order]
    first = torch.ones_like(grp, dtype=torch.bool)
    g_sorted, perm = torch.sort(grp, stable=True)
    first_s = torch.ones_like(g_sorted, dtype=torch.bool)
    first_s[1:] = g_sorted[1:] != g_sorted[:-1]
    first[perm] = first_s
    nearest_rows = rows[order][first & empty[grp]]
    if M0 > k:   # truncated: the first k empty niches in shuffled reference order take their nearest
        pos_ref = st["pos_ref"].long()
        nn = pi[nearest_rows]
        keep = torch.argsort(pos_ref[nn])[:k]
        want = torch.zeros_like(prom)
        want[nearest_rows[keep]] = True
        out["nearest_truncated"] = bool(torch.equal(want, prom))
        out["nearest_count"] = info["nearest"] == k
        return out
    out["nearest_count"] = info["nearest"] == M0
    out["nearest_promoted"] = bool(prom[nearest_rows].all())
    rho_post = rho0 + empty.long()
    rhop_post = rhop0 - empty.long()
    out["rho_post_nearest"] = bool(torch.equal(rho_post, st["rho"].long()))
    out["rho_prime_post_nearest"] = bool(torch.equal(rhop_post, st["rho_p"].long()))
    take = st["take"].long()
    per_point = torch.bincount(pi[prom], minlength=w)[:w]
    out["takes_per_point"] = bool(torch.equal(per_point, empty.long() + take))
    out["takes_total"] = int(take.sum()) == k - M0
    L = info["level"]
    lo = torch.clamp(L - rho_post, min=0)
    lo = torch.minimum(lo, rhop_post)
    hi = torch.minimum(torch.clamp(L + 1 - rho_post, min=0), rhop_post)
    out["water_level"] = bool(((take >= lo) & (take <= hi)).all())
    # cache order: among the non-nearest F_l members of a point, exactly the take_j lowest positions
    is_near = torch.zeros_like(prom)
    is_near[nearest_rows] = True
    cm = torch.nonzero(Fl & ~is_near).flatten()
    kk = pi[cm] * (R + 1) + pos[cm]
    o = torch.argsort(kk)
    gp = pi[cm][o]
    start = torch.zeros(w + 1, dtype=torch.long, device=gp.device)
    start[1:] = torch.cumsum(torch.bincount(gp, minlength=w)[:w], 0)
    idx = torch.arange(gp.numel(), device=gp.device) - start[gp]
    out["cache_order"] = bool(torch.equal(prom[cm][o], idx < take[gp]))
    return out
