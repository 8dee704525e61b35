"""Masked batch primitives (oracle; TEST INFRASTRUCTURE ONLY).  SPEC.md:22-97."""
from dataclasses import dataclass, field

import numpy as np

from paper_2504_06067_b200.errors import BoundsError, EmptySelectionError, ShapeError
from . import rng as _rng


@dataclass
class MaskedMatrix:
    """Fixed-shape data + per-row validity."""
    data: np.ndarray
    valid: np.ndarray = None

    def __post_init__(self):
        self.data = np.asarray(self.data)
        if self.valid is None:
            self.valid = np.ones(self.data.shape[0], dtype=bool)
        self.valid = np.asarray(self.valid, dtype=bool)
        if self.valid.shape != (self.data.shape[0],):
            raise ShapeError("valid must have one flag per row")


@dataclass
class SeedableRng:
    """Counter-based RNG handle: (seed, stream, epoch)."""
    seed: int
    stream: int = 0
    epoch: int = 0
    _next: int = field(default=0, repr=False)


def step_mask(x):
    """Heaviside: 1 where x > 0."""
    return (np.asarray(x) > 0).astype(np.int8)


def masked_argmin(values, valid=None):
    """Index of the minimum valid slot, lowest index on ties."""
    values = np.asarray(values)
    valid = np.ones(values.shape[0], bool) if valid is None else np.asarray(valid, bool)
    if valid.shape != values.shape:
        raise ShapeError("values/valid length mismatch")
    if not valid.any():
        raise EmptySelectionError("masked_argmin over zero valid slots")
    idx = np.flatnonzero(valid)
    return int(idx[np.argmin(values[idx])])  # argmin returns the first minimum


def segment_count(labels, valid, segments):
    """Histogram of valid labels over [0, segments)."""
    labels = np.asarray(labels, dtype=np.int64)
    valid = np.ones(labels.shape[0], bool) if valid is None else np.asarray(valid, bool)
    lab = labels[valid]
    if lab.size and (lab.min() < 0 or lab.max() >= segments):
        raise BoundsError("label out of range")
    return np.bincount(lab, minlength=segments).astype(np.int64)


def shuffle_rows(m, rng_handle):
    """Uniform row permutation; perm maps new index -> old index."""
    n = m.data.shape[0]
    perm = _rng.permutation(n, rng_handle.seed, rng_handle.epoch, rng_handle.stream)
    return MaskedMatrix(m.data[perm], m.valid[perm]), perm
