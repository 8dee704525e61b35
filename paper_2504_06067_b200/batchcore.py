"""Masked batch primitives as device tensor ops.

These are the reference's L1 building blocks; inside the engine they exist
only fused into the kernels (warp argmin reductions, warp-aggregated
histograms, keyed shuffles).  The standalone versions below keep the
reference API for callers and tests: shuffles run the library's keyed
swap-or-not kernel, the reductions are single device tensor expressions.
"""
from dataclasses import dataclass

import torch

from . import _lib
from ._tensor import as_cuda
from .errors import BoundsError, EmptySelectionError, ShapeError


@dataclass
class MaskedMatrix:
    """Fixed-shape rows + validity flags."""
    data: torch.Tensor
    valid: torch.Tensor = None

    def __post_init__(self):
        self.data = as_cuda(self.data, torch.float32) if not isinstance(self.data, torch.Tensor) else self.data
        if self.valid is None:
            self.valid = torch.ones(self.data.shape[0], dtype=torch.bool, device=self.data.device)
        self.valid = as_cuda(self.valid, torch.bool)
        if self.valid.shape != (self.data.shape[0],):
            raise ShapeError("valid must have one flag per row")


@dataclass
class SeedableRng:
    """Counter-based RNG handle: Philox key = seed, counter words (idx, epoch, stream)."""
    seed: int
    stream: int = 0
    epoch: int = 0


def step_mask(x):
    """Heaviside H(x) = 1 where x > 0."""
    return (as_cuda(x, torch.float32) > 0).to(torch.int8)


def masked_argmin(values, valid=None):
    """Lowest-index minimum over valid slots."""
    v = as_cuda(values, torch.float64)
    ok = torch.ones_like(v, dtype=torch.bool) if valid is None else as_cuda(valid, torch.bool)
    if ok.shape != v.shape:
        raise ShapeError("values/valid length mismatch")
    if not bool(ok.any()):
        raise EmptySelectionError("masked_argmin over zero valid slots")
    masked = torch.where(ok, v, torch.full_like(v, float("inf")))
    mn = masked.min()
    hit = ok & (masked == mn)
    return int(torch.nonzero(hit)[0, 0].item())


def segment_count(labels, valid, segments):
    """Count of valid labels per segment."""
    lab = as_cuda(labels, torch.int64)
    ok = torch.ones_like(lab, dtype=torch.bool) if valid is None else as_cuda(valid, torch.bool)
    lab = lab[ok]
    if lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= segments):
        raise BoundsError("label out of range")
    return torch.bincount(lab, minlength=segments)


def shuffle_rows(m, rng):
    """Uniformly permuted rows + permutation (new index -> old index)."""
    n = m.data.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=m.data.device)
    if n:
        _lib.check(_lib.lib().mo_permutation(n, int(rng.seed), int(rng.epoch), int(rng.stream), _lib.ptr(perm),
                                             _lib.ptr(None), _lib.stream_ptr()), "mo_permutation")
    p = perm.long()
    return MaskedMatrix(m.data[p], m.valid[p]), perm
