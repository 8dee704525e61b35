"""Mating pool + SBX + polynomial mutation (+ fused DTLZ evaluation) on the GPU.

SPEC.md:238-308.  The production operator is :func:`vary_eval`, one fused
kernel (``k_vary_eval``): keyed mating permutation -> SBX -> clamp -> PM ->
clamp -> DTLZ, with the Philox streams of DESIGN.md.
"""
from dataclasses import dataclass

import torch

from . import _lib
from ._tensor import as_matrix
from .errors import ParameterError, ShapeError

STREAM_INIT, STREAM_MATING, STREAM_SBX, STREAM_PM, STREAM_POP_SHUFFLE, STREAM_REF_SHUFFLE = 1, 2, 3, 4, 5, 6


@dataclass(frozen=True)
class VariationConfig:
    """SPEC.md:243-246; defaults SPEC.md:293 (p_m=None means 1/d)."""
    eta_c: float = 20.0
    eta_m: float = 20.0
    p_c: float = 1.0
    p_m: float = None

    def __post_init__(self):
        if not (self.eta_c > 0 and self.eta_m > 0):
            raise ParameterError("eta_c and eta_m must be > 0")
        if not (0.0 <= self.p_c <= 1.0) or (self.p_m is not None and not 0.0 <= self.p_m <= 1.0):
            raise ParameterError("probabilities must lie in [0,1]")

    def c_struct(self):
        return _lib.VarCfg(self.eta_c, self.eta_m, self.p_c, -1.0 if self.p_m is None else self.p_m)


def permutation(n, seed, generation, stream):
    """perm[p] = item at shuffled position p (int32 CUDA tensor), keyed swap-or-not."""
    perm = torch.empty(int(n), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().mo_permutation(int(n), int(seed), int(generation), int(stream), _lib.ptr(perm),
                                         _lib.ptr(None), _lib.stream_ptr()), "mo_permutation")
    return perm


def mating_pool(n, seed, generation):
    """(n/2, 2) parent pairs: a keyed permutation split into consecutive pairs."""
    if n % 2:
        raise ParameterError("mating pool needs even n")
    return permutation(n, seed, generation, STREAM_MATING).view(-1, 2)


def vary_eval(problem, X, cfg, seed, generation, ideal=None):
    """Offspring (n x d) and their objectives (n x m) from parents X (n x d).

    If ``ideal`` (m FP32 CUDA tensor) is given it is lowered in place to the
    offspring column minima.
    """
    X = as_matrix(X)
    n, d = X.shape
    if d != problem.d:
        raise ShapeError("X must be n x d")
    if n % 2:
        raise ParameterError("variation needs even n")
    Xo = torch.empty_like(X)
    Fo = torch.empty((n, problem.m), dtype=torch.float32, device=X.device)
    c = cfg.c_struct()
    _lib.check(_lib.lib().mo_vary_eval(problem.id, _lib.ptr(X), n, d, problem.m, int(seed), int(generation),
                                       c, _lib.ptr(Xo), _lib.ptr(Fo), _lib.ptr(ideal), _lib.stream_ptr()),
               "mo_vary_eval")
    return Xo, Fo


def init_population(n, d, seed):
    """engine.initialize's uniform population in [0,1]^d, FP32 CUDA tensor."""
    X = torch.empty((int(n), int(d)), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().mo_init_population(_lib.ptr(X), int(n), int(d), int(seed), _lib.stream_ptr()),
               "mo_init_population")
    return X
