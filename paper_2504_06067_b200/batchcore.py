"""Masked batch primitives as device tensor ops.

These are the reference's L1 building blocks; inside the engine they exist
only fused into the kernels (warp argmin reductions, warp-aggregated
histograms, keyed shuffles).  The standalone versions below keep the
reference API for callers and tests: shuffles run the library's keyed
swap-or-not kernel, step_mask / masked_argmin / segment_count their own small
kernels (k_ops.cu).
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
    """Heaviside H(x) = 1 where x > 0; int8 CUDA tensor (k_step_mask)."""
    x = as_cuda(x, torch.float64).reshape(-1)
    out = torch.empty(x.numel(), dtype=torch.int8, device=x.device)
    _lib.check(_lib.lib().mo_step_mask(_lib.ptr(x), x.numel(), _lib.ptr(out), _lib.stream_ptr()), "mo_step_mask")
    return out


def masked_argmin(values, valid=None):
    """Lowest-index minimum over valid slots; EmptySelectionError when none is valid."""
    v = as_cuda(values, torch.float64).reshape(-1)
    ok = None if valid is None else as_cuda(valid, torch.uint8).reshape(-1)
    if ok is not None and ok.shape != v.shape:
        raise ShapeError("values/valid length mismatch")
    out = torch.empty(1, dtype=torch.int64, device=v.device)
    ws = _lib.workspace_ops(v.numel(), 1, v.device)
    _lib.check(_lib.lib().mo_masked_argmin(_lib.ptr(v), _lib.ptr(ok), v.numel(), _lib.ptr(out), _lib.ptr(ws),
                                           ws.numel(), _lib.stream_ptr()), "mo_masked_argmin")
    i = int(out.item())
    if i < 0:
        raise EmptySelectionError("masked_argmin over zero valid slots")
    return i


def segment_count(labels, valid, segments):
    """Count of valid labels per segment; BoundsError for a valid label out of range."""
    lab = as_cuda(labels, torch.int64).reshape(-1)
    ok = None if valid is None else as_cuda(valid, torch.uint8).reshape(-1)
    if ok is not None and ok.shape != lab.shape:
        raise ShapeError("labels/valid length mismatch")
    counts = torch.empty(int(segments), dtype=torch.int64, device=lab.device)
    status = torch.zeros(1, dtype=torch.int32, device=lab.device)
    _lib.check(_lib.lib().mo_segment_count(_lib.ptr(lab), _lib.ptr(ok), lab.numel(), int(segments), _lib.ptr(counts),
                                           _lib.ptr(status), _lib.stream_ptr()), "mo_segment_count")
    if int(status.item()):
        raise BoundsError("label out of range")
    return counts


def shuffle_rows(m, rng):
    """Uniformly permuted rows + permutation (new index -> old index)."""
    n = m.data.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=m.data.device)
    if n:
        _lib.check(_lib.lib().mo_permutation(n, int(rng.seed), int(rng.epoch), int(rng.stream), _lib.ptr(perm),
                                             _lib.ptr(None), _lib.stream_ptr()), "mo_permutation")
    p = perm.long()
    return MaskedMatrix(m.data[p], m.valid[p]), perm
