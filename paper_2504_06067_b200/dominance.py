"""Pareto dominance and non-dominated sorting on the GPU.

``dominance_matrix`` / ``non_dominated_sort`` / ``split_fronts`` keep the
reference signatures; the work runs in ``k_dom_tile`` (warp-ballot bit-matrix)
and ``k_front_peel`` (persistent resume-scan peeling) of libmanyobj_b200.so.
"""
from dataclasses import dataclass

import torch

from . import _lib
from ._tensor import as_cuda, as_mask, as_matrix, device
from .errors import InfeasibleSplitError, ParameterError, ShapeError

DROPPED = _lib.DROPPED


def dominates(a, b):
    """a <= b everywhere and a < b somewhere."""
    a = as_cuda(a, torch.float32)
    b = as_cuda(b, torch.float32)
    if a.shape != b.shape:
        raise ShapeError("objective vectors differ in length")
    return bool(((a <= b).all() & (a < b).any()).item())


def dominance_bits(F, valid=None):
    """Raw bit-matrix: (R x W) int32 words, bit i of row j = "F[i] dominates F[j]"."""
    F = as_matrix(F)
    R, m = F.shape
    W = int(_lib.lib().mo_bits_words_per_row(R))
    bits = torch.empty((R, W), dtype=torch.int32, device=F.device)
    v = as_mask(valid, R)
    _lib.check(_lib.lib().mo_dominance_bits(_lib.ptr(F), R, m, _lib.ptr(v), _lib.ptr(bits), _lib.stream_ptr()),
               "mo_dominance_bits")
    return bits


def presort(F):
    """The engine's sort-path prologue: rows bucketed by S = FP32 left-to-right objective sum.

    Returns a dict of CUDA tensors: perm[p] = row at position p (buckets in
    S order, arbitrary order inside a bucket), FS / SS = rows / sums in that
    order, wend[p] = one past the last bit-matrix word that can hold a
    dominator of p, blkmin / blkmax = S range of every 256-position block.
    """
    F = as_matrix(F)
    R, m = F.shape
    dev = F.device
    nb = (R + 255) // 256
    out = dict(perm=torch.empty(R, dtype=torch.int32, device=dev), FS=torch.empty_like(F),
               SS=torch.empty(R, dtype=torch.float32, device=dev), wend=torch.empty(R, dtype=torch.int32, device=dev),
               blkmin=torch.empty(nb, dtype=torch.float32, device=dev),
               blkmax=torch.empty(nb, dtype=torch.float32, device=dev))
    ws = _lib.workspace_rows(R, m, 1, dev)
    _lib.check(_lib.lib().mo_presort(_lib.ptr(F), R, m, *(_lib.ptr(out[k]) for k in
                                                          ("perm", "FS", "SS", "wend", "blkmin", "blkmax")),
                                     _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "mo_presort")
    return out


def dominance_bits_sorted(ps, poison=False, method="ranked", summary=None):
    """Bit-matrix of presorted rows (position space) + has-a-dominator flags, from :func:`presort`.
    ``method``: "ranked" (per-objective rank masks, k_dom_rank.cu -- the engine's kernel) or
    "pairwise" (compare-chain tiles, k_dom_tile_sorted).  ``poison`` pre-fills the matrix with ones
    (tests: words below wend must all be written).  ``summary``: an int32 tensor of R x
    mo_tile_summary_words(R) words receiving the engine's tile summary (ranked only; then only nonzero
    256-bit word blocks are stored)."""
    FS = ps["FS"]
    R, m = FS.shape
    L = _lib.lib()
    W = int(L.mo_bits_words_per_row(R))
    bits = torch.full((R, W), -1 if poison else 0, dtype=torch.int32, device=FS.device)
    hasdom = torch.empty(R, dtype=torch.uint8, device=FS.device)
    args = (_lib.ptr(FS), _lib.ptr(ps["blkmin"]), _lib.ptr(ps["blkmax"]), _lib.ptr(ps["wend"]), R, m,
            _lib.ptr(bits), _lib.ptr(hasdom))
    if method == "ranked":
        nbytes = int(L.mo_dominance_tables_bytes(R, m))
        if nbytes == 0:
            raise ParameterError("the rank-mask kernel needs 2 <= m <= 512")
        tables = torch.empty(nbytes, dtype=torch.uint8, device=FS.device)
        _lib.check(L.mo_dominance_bits_ranked(*args, _lib.ptr(tables), nbytes,
                                              _lib.ptr(summary) if summary is not None else None,
                                              _lib.stream_ptr()), "mo_dominance_bits_ranked")
    elif method == "pairwise":
        _lib.check(L.mo_dominance_bits_sorted(*args, _lib.stream_ptr()), "mo_dominance_bits_sorted")
    else:
        raise ParameterError(f"unknown method {method!r}")
    return bits, hasdom


def unpack_bits(bits, R):
    """(R x W) words -> dense bool M with M[i][j] = bit i of row j."""
    w = bits.view(torch.int32)
    shifts = torch.arange(32, device=w.device, dtype=torch.int32)
    b = ((w.unsqueeze(-1) >> shifts) & 1).bool()          # rows j, words, bit -> i
    dom_of = b.reshape(w.shape[0], -1)[:, :R]              # [j, i]
    return dom_of.t().contiguous()                         # [i, j]


def dominance_matrix(F, valid=None):
    """M[i][j] = dominates(F[i], F[j]) as a bool CUDA tensor."""
    F = as_matrix(F)
    return unpack_bits(dominance_bits(F, valid), F.shape[0])


def non_dominated_sort(F, valid=None, stop_at=None, return_info=False):
    """Front index per row; invalid / beyond-split rows -> DROPPED.

    ``stop_at`` (the engine's n) stops peeling at the first front whose
    cumulative size reaches it.  Returns an int32 CUDA tensor.
    """
    F = as_matrix(F)
    R, m = F.shape
    if R == 0:
        raise ShapeError("need at least one row")
    bits = dominance_bits(F, valid)
    v = as_mask(valid, R)
    ranks = torch.empty(R, dtype=torch.int32, device=F.device)
    info = _lib.new_info(F.device)
    ws = _lib.workspace_rows(R, m, 1, F.device)
    L = _lib.lib()
    _lib.check(L.mo_front_peel(_lib.ptr(bits), R, _lib.ptr(v), int(stop_at or 0), _lib.ptr(ranks), _lib.ptr(info),
                               _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "mo_front_peel")
    if return_info:
        return ranks, info
    return ranks


def stream_sort(F, n, shards=1, poll=1):
    """non_dominated_sort + split_fronts of R = 2n rows through the streamed
    (no bit-matrix) sort the engine uses when the bit-matrix exceeds HBM and
    when it shards (mo_sort_stream_*).  ``shards`` > 1 runs every shard in
    this process on its own workspace and exchanges the front masks by
    concatenation -- the same bytes NCCL's all-gather moves between GPUs.
    Returns (ranks, info) of shard 0 (all shards agree; checked)."""
    F = as_matrix(F)
    R, m = F.shape
    if R != 2 * n or n < 1:
        raise ShapeError("stream_sort needs R = 2n rows")
    L = _lib.lib()
    s = _lib.stream_ptr()
    nb = _lib.workspace_bytes_ex(n, m, m, 1, _lib.SORT_STREAM, shards)
    lo, words, fo, _ = _lib.stream_offsets(n, m, 1, _lib.SORT_STREAM, shards)
    shard = []
    for g in range(shards):
        ws = torch.empty(nb, dtype=torch.uint8, device=F.device)
        ranks = torch.empty(R, dtype=torch.int32, device=F.device)
        info = _lib.new_info(F.device)
        a = _lib.StepArgs()
        a.problem, a.m, a.d, a.n, a.w = 1, m, m, n, 1
        for f in ("zhat", "XR", "FR", "X_next", "F_next", "ideal"):
            setattr(a, f, F.data_ptr())
        a.ranks, a.info = ranks.data_ptr(), info.data_ptr()
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
        a.sort_mode, a.shard_rank, a.shard_count = _lib.SORT_STREAM, g, shards
        loc = ws[lo: lo + 4 * words].view(torch.int32)
        full = ws[fo: fo + 4 * words * shards].view(torch.int32)
        shard.append((a, ranks, info, loc, full))
        _lib.check(L.mo_sort_stream_begin(a, s), "mo_sort_stream_begin")
    k = 0
    while True:
        if shards > 1:
            cat = torch.cat([x[3] for x in shard])
            for x in shard:
                x[4].copy_(cat)
        for x in shard:
            _lib.check(L.mo_sort_stream_front(x[0], k, s), "mo_sort_stream_front")
        k += 1
        if k % poll == 0 and int(shard[0][2][_lib.INFO["NFRONTS"]].item()) > 0:
            break
    for x in shard:
        _lib.check(L.mo_sort_stream_end(x[0], s), "mo_sort_stream_end")
    for x in shard[1:]:
        if not (torch.equal(x[1], shard[0][1]) and torch.equal(x[2], shard[0][2])):
            raise RuntimeError("shards disagree on the ranks")
    return shard[0][1], shard[0][2]


@dataclass(frozen=True)
class FrontSplit:
    """SPEC.md:172-175."""
    l: int
    selected_count: int
    k: int


def split_fronts(ranks, n):
    """l / selected_count / k of a rank vector."""
    r = as_cuda(ranks, torch.int64)
    live = r[r != DROPPED]
    if live.numel() < n:
        raise InfeasibleSplitError(f"{live.numel()} valid individuals < n={n}")
    sizes = torch.bincount(live)
    cum = torch.cumsum(sizes, 0)
    l = int(torch.searchsorted(cum, torch.tensor([n], device=cum.device)).item())
    sel = int(cum[l - 1].item()) if l > 0 else 0
    return FrontSplit(l, sel, n - sel)


def split_from_info(info):
    """FrontSplit from the device info record written by mo_front_peel / mo_step."""
    h = info.cpu().tolist()
    err = h[_lib.INFO["ERROR"]]
    if err:
        _lib.check(err, "front peeling")
    return FrontSplit(h[_lib.INFO["L"]], h[_lib.INFO["SELECTED"]], h[_lib.INFO["K"]])


__all__ = ["DROPPED", "dominates", "dominance_bits", "dominance_matrix", "non_dominated_sort", "FrontSplit",
           "split_fronts", "split_from_info", "unpack_bits", "presort", "dominance_bits_sorted", "device", "stream_sort"]
