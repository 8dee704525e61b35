"""NSGA-III niching: Alg. 2 batched back-end + Alg. 1 scalar oracle.

TEST INFRASTRUCTURE ONLY.  Restates SPEC.md:310-433 (niche module) and
PAPER.md:157-191 (Alg. 2) / PAPER.md:107-134 (Alg. 1), with DESIGN.md's pins:

* normalisation (A-4): FP32 running-min ideal over all 2n
  rows; ASF extremes over rows with rank <= l (ties -> lowest shuffled
  population position); FP64 Gaussian elimination with partial pivoting for
  the hyperplane, every op separately rounded; per-component fallback to the
  max translated value, then 1; Fn = FP32(f - ideal) / FP32(a).
* association (A-2): canonical FP32 key
  t_j = ((f0*z0 + f1*z1) + ...) with zhat = z/||z||, pi = argmax t with the
  lowest *shuffled* reference position on ties, d = sqrt(sum_k (f_k - t*z_k)^2)
  left to right.  Equal to argmin of ||f|| sqrt(1 - cos^2) in real arithmetic.
* every "lowest index" tie-break uses shuffled positions (A-5); the cache
  excludes nearest-taken candidates and cursors start at 0 (A-6); promoted
  individuals get rank l-1 (A-8).
"""
import numpy as np

from paper_2504_06067_b200.errors import EmptySelectionError, InfeasibleSplitError
from . import rng as _rng
from .dominance import DROPPED

INF = np.int64(2 ** 31 - 1)
ASF_EPS = np.float32(1e-6)
DEGENERATE = 1e-10


# ----------------------------------------------------------- normalisation

def gauss_solve(E):
    """Solve E b = 1 (m x m, float64) with partial pivoting; None if singular."""
    m = len(E)
    A = [[float(v) for v in row] for row in E]
    rhs = [1.0] * m
    for c in range(m):
        p = c
        best = abs(A[c][c])
        for r in range(c + 1, m):
            if abs(A[r][c]) > best:
                best = abs(A[r][c])
                p = r
        if best == 0.0:
            return None
        if p != c:
            A[c], A[p] = A[p], A[c]
            rhs[c], rhs[p] = rhs[p], rhs[c]
        for r in range(c + 1, m):
            f = A[r][c] / A[c][c]
            for cc in range(c, m):
                A[r][cc] = A[r][cc] - f * A[c][cc]
            rhs[r] = rhs[r] - f * rhs[c]
    b = [0.0] * m
    for c in reversed(range(m)):
        s = rhs[c]
        for cc in range(c + 1, m):
            s = s - A[c][cc] * b[cc]
        b[c] = s / A[c][c]
    return b


def extreme_points(Ft, cand, pos_pop):
    """Row index of the ASF-minimal candidate for every axis."""
    m = Ft.shape[1]
    rows = np.flatnonzero(cand)
    order = rows[np.argsort(pos_pop[rows], kind="stable")]     # shuffled order
    sub = Ft[order]
    out = []
    for a in range(m):
        w = np.full(m, ASF_EPS, dtype=np.float32)
        w[a] = np.float32(1.0)
        asf = (sub / w[None, :]).max(axis=1)                      # FP32 division, max
        out.append(int(order[int(np.argmin(asf))]))                # first min = lowest pos
    return out


def intercepts(Ft, cand, ext):
    m = Ft.shape[1]
    fallback = []
    mx = Ft[cand].max(axis=0).astype(np.float64)
    for k in range(m):
        fallback.append(float(mx[k]) if mx[k] > DEGENERATE else 1.0)
    b = gauss_solve(Ft[ext].astype(np.float64))
    if b is None or not all(np.isfinite(v) for v in b):
        return np.array(fallback), True
    a = []
    for k in range(m):
        ak = 1.0 / b[k]
        a.append(ak if (np.isfinite(ak) and ak > DEGENERATE) else fallback[k])
    return np.array(a), False


def normalize_objectives(F, ideal_prev, cand, pos_pop):
    """(Fn FP32, ideal FP32, a FP64, extremes, singular) -- SPEC.md:331-339."""
    F = np.asarray(F, dtype=np.float32)
    ideal = np.minimum(np.asarray(ideal_prev, np.float32), F.min(axis=0))
    Ft = F - ideal[None, :]
    ext = extreme_points(Ft, cand, pos_pop)
    a, singular = intercepts(Ft, cand, ext)
    Fn = Ft / a.astype(np.float32)[None, :]
    return Fn, ideal, a, ext, singular


def normalize_spec(F, ideal=None):
    """SPEC.md:331-339 in float64 with all rows as candidates (for the KATs)."""
    F = np.asarray(F, dtype=np.float64)
    ideal = F.min(axis=0) if ideal is None else np.minimum(ideal, F.min(axis=0))
    Ft = F - ideal
    m = F.shape[1]
    ext = []
    for a_ in range(m):
        w = np.full(m, 1e-6)
        w[a_] = 1.0
        ext.append(int(np.argmin((Ft / w).max(axis=1))))
    cand = np.ones(F.shape[0], bool)
    a, _ = intercepts(Ft, cand, ext)
    return Ft / a, ideal, a


# ------------------------------------------------------------- association

def perpendicular_distance_matrix(Fn, Z):
    """D[i][j] = ||f_i|| sqrt(1 - cos^2 theta_ij) (float64).

    Evaluated as the length of the rejection ||f - (f . zhat) zhat||, the same
    quantity without the cancellation of 1 - cos^2 (the literal form is off by
    ~1e-8 for near-parallel pairs and would fail SPEC.md:410/:729's 1e-9
    agreement with direct projection).  f = 0 gives a row of zeros.
    """
    Fn = np.asarray(Fn, np.float64)
    Z = np.asarray(Z, np.float64)
    zn = np.sqrt((Z * Z).sum(axis=1))
    if (zn == 0).any():
        from paper_2504_06067_b200.errors import ParameterError
        raise ParameterError("zero reference point")
    zh = Z / zn[:, None]
    t = Fn @ zh.T                                        # (R, w) projections
    E = Fn[:, None, :] - t[:, :, None] * zh[None, :, :]  # (R, w, m) rejections
    return np.sqrt((E * E).sum(axis=2))


def perpendicular_distance_literal(Fn, Z):
    """The literal ||f|| sqrt(1 - cos^2) form of SPEC.md:343 (cos clamped, f=0 -> 0)."""
    Fn = np.asarray(Fn, np.float64)
    Z = np.asarray(Z, np.float64)
    fn = np.sqrt((Fn * Fn).sum(axis=1))
    zn = np.sqrt((Z * Z).sum(axis=1))
    with np.errstate(invalid="ignore", divide="ignore"):
        cos = (Fn @ Z.T) / (fn[:, None] * zn[None, :])
    cos = np.clip(np.nan_to_num(cos, nan=1.0), -1.0, 1.0)
    D = fn[:, None] * np.sqrt(1.0 - cos * cos)
    D[fn == 0] = 0.0
    return D


def associate(D, valid=None):
    """argmin per valid row, lowest index on ties; invalid rows -> (-1, nan)."""
    D = np.asarray(D)
    valid = np.ones(D.shape[0], bool) if valid is None else np.asarray(valid, bool)
    pi = np.full(D.shape[0], -1, dtype=np.int64)
    d = np.full(D.shape[0], np.nan)
    pi[valid] = np.argmin(D[valid], axis=1)
    d[valid] = D[valid, pi[valid]]
    return pi, d


def associate_canonical(Fn, zhat, pos_ref, rows, block=512):
    """Canonical FP32 association of ``rows`` (index array) -> (pi, d) full-length."""
    Fn = np.asarray(Fn, np.float32)
    zhat = np.asarray(zhat, np.float32)
    w, m = zhat.shape
    perm_ref = np.empty(w, np.int64)
    perm_ref[pos_ref] = np.arange(w)
    zs = zhat[perm_ref]                      # refs in shuffled order
    R = Fn.shape[0]
    pi = np.full(R, -1, np.int64)
    d = np.full(R, np.nan, np.float32)
    for b0 in range(0, len(rows), block):
        rr = rows[b0:b0 + block]
        f = Fn[rr]
        t = f[:, 0, None] * zs[None, :, 0]
        for k in range(1, m):
            t = t + f[:, k, None] * zs[None, :, k]
        p = np.argmax(t, axis=1)             # first maximum = lowest shuffled position
        tb = t[np.arange(len(rr)), p]
        zb = zs[p]
        e = f[:, 0] - tb * zb[:, 0]
        s = e * e
        for k in range(1, m):
            e = f[:, k] - tb * zb[:, k]
            s = s + e * e
        pi[rr] = perm_ref[p]
        d[rr] = np.sqrt(s)
    return pi, d


# ------------------------------------------------------------ niche counts

def niche_counts(pi, ranks, l, w):
    """rho over rank<l, rho' over rank==l, rho=INF where rho'==0."""
    pi = np.asarray(pi)
    ranks = np.asarray(ranks)
    sel = (ranks < l) & (ranks != DROPPED) if l > 0 else np.zeros(len(ranks), bool)
    rho = np.bincount(pi[sel], minlength=w).astype(np.int64)
    rho_p = np.bincount(pi[ranks == l], minlength=w).astype(np.int64)
    rho[rho_p == 0] = INF
    return rho, rho_p


def _first_k_by_pos(js, k, pos_ref):
    js = np.asarray(js)
    if len(js) <= k:
        return js
    return js[np.argsort(pos_ref[js], kind="stable")][:k]


def nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref):
    """Alg. 2 lines 8-12.  Returns (promoted rows, rho, rho_p)."""
    rho = rho.copy()
    rho_p = rho_p.copy()
    empty = np.flatnonzero(rho == 0)
    if len(empty) == 0 or k <= 0:
        return np.zeros(0, np.int64), rho, rho_p
    fl = np.flatnonzero(ranks == l)
    chosen = {}
    for j in empty:
        cand = fl[pi[fl] == j]
        key = np.lexsort((pos_pop[cand], d[cand]))        # d first, then position
        chosen[int(j)] = int(cand[key[0]])
    kept = _first_k_by_pos(empty, k, pos_ref)
    promoted = np.array([chosen[int(j)] for j in kept], dtype=np.int64)
    rho[kept] = 1
    rho_p[kept] -= 1
    rho[rho_p == 0] = INF
    return promoted, rho, rho_p


def nearest_selection_vec(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref):
    """:func:`nearest_selection` without the per-point loop (one lexsort; O(R log R)): the same
    promoted rows and counts (tests/test_oracle_fast.py), for the checker at C2-C4 sizes where the
    loop's per-point scans of F_l are quadratic."""
    rho = rho.copy()
    rho_p = rho_p.copy()
    empty = np.flatnonzero(rho == 0)
    if len(empty) == 0 or k <= 0:
        return np.zeros(0, np.int64), rho, rho_p
    fl = np.flatnonzero(ranks == l)
    is_empty = np.zeros(len(rho), bool)
    is_empty[empty] = True
    c = fl[is_empty[pi[fl]]]
    c = c[np.lexsort((pos_pop[c], d[c], pi[c]))]            # per point: d first, then position
    pc = pi[c]
    first = np.ones(len(c), bool)
    first[1:] = pc[1:] != pc[:-1]
    chosen = np.full(len(rho), -1, np.int64)
    chosen[pc[first]] = c[first]
    kept = _first_k_by_pos(empty, k, pos_ref)
    promoted = chosen[kept].astype(np.int64)
    rho[kept] = 1
    rho_p[kept] -= 1
    rho[rho_p == 0] = INF
    return promoted, rho, rho_p


def build_cache(pi, ranks, l, w, pos_pop, exclude):
    """Per reference point, F_l candidates in shuffled population order.

    Returned as CSR (offsets[w+1], cand) -- the dense w x |F_l| table of the
    paper is the same rows without sentinel padding.
    """
    fl = np.flatnonzero(ranks == l)
    fl = fl[~np.isin(fl, exclude)]
    order = fl[np.lexsort((pos_pop[fl], pi[fl]))]
    counts = np.bincount(pi[order], minlength=w)
    offsets = np.zeros(w + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    return offsets, order


def batched_random_selection(offsets, cand, rho, rho_p, k, pos_ref):
    """Alg. 2 lines 15-26 loop.  Returns (promoted rows, iterations)."""
    rho = rho.copy()
    rho_p = rho_p.copy()
    cursor = np.zeros(len(rho), np.int64)
    taken = []
    it = 0
    while k > 0:
        finite = rho < INF
        if not finite.any():
            raise InfeasibleSplitError("niche loop cannot progress")
        mn = rho[finite].min()
        u = np.flatnonzero(rho == mn)
        u = _first_k_by_pos(u, k, pos_ref)
        for j in u:
            taken.append(int(cand[offsets[j] + cursor[j]]))
        cursor[u] += 1
        rho[u] += 1
        rho_p[u] -= 1
        rho[rho_p == 0] = INF
        k -= len(u)
        it += 1
    return np.array(taken, np.int64), it


def waterfill_takes(rho, rho_p, k, pos_ref):
    """Closed form of the loop: number of cache entries each point takes.

    After the nearest pass every active point j has finite rho_j and c_j =
    rho'_j candidates; at level L a point is marked iff rho_j <= L < rho_j + c_j.
    T(L) = sum_j clamp(L + 1 - rho_j, 0, c_j) takes are done once level L is
    processed; L* = min{L : T(L) >= k}; the last level is truncated to the
    first k - T(L*-1) marked points in shuffled reference order.
    """
    take = np.zeros(len(rho), np.int64)
    if k <= 0:
        return take
    act = rho < INF
    if not act.any():
        raise InfeasibleSplitError("niche loop cannot progress")
    r = rho[act]
    c = rho_p[act]

    def T(L):
        return int(np.clip(L + 1 - r, 0, c).sum())

    lo, hi = int(r.min()), int((r + c).max())
    if T(hi) < k:
        raise InfeasibleSplitError("not enough candidates")
    while lo < hi:
        mid = (lo + hi) // 2
        if T(mid) >= k:
            hi = mid
        else:
            lo = mid + 1
    L = lo
    base = np.clip(L - r, 0, c)
    need = k - int(base.sum())
    idx = np.flatnonzero(act)
    take[idx] = base
    marked = idx[(r <= L) & (L < r + c)]
    keep = _first_k_by_pos(marked, need, pos_ref)
    take[keep] += 1
    return take


def waterfill_selection(offsets, cand, rho, rho_p, k, pos_ref):
    take = waterfill_takes(rho, rho_p, k, pos_ref)
    out = [cand[offsets[j]:offsets[j] + take[j]] for j in np.flatnonzero(take)]
    return np.concatenate(out) if out else np.zeros(0, np.int64)


# ------------------------------------------------------------ Alg. 1 oracle

def oracle_niche_select(pi, d, ranks, l, k, w, gen):
    """Alg. 1 lines 7-19 one point at a time.  ``gen``: numpy Generator."""
    ranks = np.asarray(ranks)
    sel_mask = (ranks < l) & (ranks != DROPPED) if l > 0 else np.zeros(len(ranks), bool)
    rho = np.bincount(pi[sel_mask], minlength=w).astype(np.int64)
    fl = list(np.flatnonzero(ranks == l))
    members = {}
    for i in fl:
        members.setdefault(int(pi[i]), []).append(int(i))
    active = np.ones(w, bool)
    out = []
    while len(out) < k:
        if not active.any():
            raise InfeasibleSplitError("oracle niche loop cannot progress")
        mn = rho[active].min()
        pts = np.flatnonzero(active & (rho == mn))
        v = int(pts[gen.integers(len(pts))])
        cands = members.get(v, [])
        if not cands:
            active[v] = False
            continue
        if rho[v] == 0:
            dv = np.array([d[i] for i in cands])
            best = np.flatnonzero(dv == dv.min())
            t = cands[int(best[gen.integers(len(best))])]
        else:
            t = cands[int(gen.integers(len(cands)))]
        cands.remove(t)
        out.append(t)
        rho[v] += 1
    return np.array(out, np.int64)


# ------------------------------------------------------------- full pipeline

def select(F, ranks, split, ideal_prev, zhat, seed, generation, backend="batched", gen=None,
           loop="waterfill", associate_fn=None, fast=False):
    """Survivor selection of Alg. 1/2 given NDS ranks.  Returns (selected mask, info).

    ``associate_fn(Fn, zhat, pos_ref, rows) -> (pi, d)`` replaces :func:`associate_canonical` (the
    C restatement in oracle/c at large sizes); ``fast`` uses :func:`nearest_selection_vec`."""
    F = np.asarray(F, np.float32)
    R = F.shape[0]
    w = zhat.shape[0]
    l, k = split.l, split.k
    ranks = np.asarray(ranks).copy()
    info = {"l": l, "k": k, "selected_count": split.selected_count}
    fl_size = int((ranks == l).sum())
    ideal = np.minimum(np.asarray(ideal_prev, np.float32), F.min(axis=0))
    info["ideal"] = ideal
    if fl_size == k:                         # cum(<=l) == n: keep all of F_l (A-3)
        info["skipped"] = True
        return (ranks <= l) & (ranks != DROPPED), info
    info["skipped"] = False
    pos_pop = _rng.positions(R, seed, generation, _rng.STREAM_POP_SHUFFLE)
    pos_ref = _rng.positions(w, seed, generation, _rng.STREAM_REF_SHUFFLE)
    cand = (ranks <= l) & (ranks != DROPPED)
    Fn, ideal, a, ext, singular = normalize_objectives(F, ideal_prev, cand, pos_pop)
    rows = np.flatnonzero(cand)
    pi, d = (associate_fn or associate_canonical)(Fn, zhat, pos_ref, rows)
    info.update(Fn=Fn, intercepts=a, extremes=ext, singular=singular, pi=pi, d=d,
                pos_pop=pos_pop, pos_ref=pos_ref)
    if backend == "oracle":
        promoted = oracle_niche_select(pi, d, ranks, l, k, w, gen or np.random.default_rng(seed))
    else:
        rho, rho_p = niche_counts(pi, ranks, l, w)
        near, rho, rho_p = (nearest_selection_vec if fast else nearest_selection)(
            pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
        k_rem = k - len(near)
        offsets, cq = build_cache(pi, ranks, l, w, pos_pop, near)
        if loop == "loop":
            rest, it = batched_random_selection(offsets, cq, rho, rho_p, k_rem, pos_ref)
            info["iterations"] = it
        else:
            rest = waterfill_selection(offsets, cq, rho, rho_p, k_rem, pos_ref)
        promoted = np.concatenate([near, rest])
        info["nearest"] = near
    sel = (ranks < l) & (ranks != DROPPED) if l > 0 else np.zeros(R, bool)
    sel = sel.copy()
    sel[promoted] = True
    info["promoted"] = promoted
    return sel, info
