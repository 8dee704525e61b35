"""Mating pool + SBX + polynomial mutation (+ fused DTLZ evaluation) on the GPU.

SPEC.md:238-308.  The production operator is :func:`vary_eval`, one fused
kernel (``k_vary_eval``): keyed mating permutation -> SBX -> clamp -> PM ->
clamp -> DTLZ, with the Philox streams of DESIGN.md.
"""
from dataclasses import dataclass

import torch

from . import _lib
from ._tensor import as_cuda, as_matrix
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


def positions(n, seed, generation, stream):
    """pos[i] = shuffled position of item i (inverse of :func:`permutation`), int64 CUDA tensor."""
    pos = torch.empty(int(n), dtype=torch.int32, device="cuda")
    perm = torch.empty(int(n), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().mo_permutation(int(n), int(seed), int(generation), int(stream), _lib.ptr(perm),
                                         _lib.ptr(pos), _lib.stream_ptr()), "mo_permutation")
    return pos.long()


def _pairs64(x):
    t = as_cuda(x, torch.float64)
    return t.reshape(1, -1) if t.ndim == 1 else t


def sbx_pair(p1, p2, u=None, eta=20.0, lo=0.0, hi=1.0, clamp=True, cfg=None, seed=0, generation=0):
    """children (c1, c2) of parent vectors p1, p2 (one pair, or a batch of pairs as
    rows), FP64.  ``u`` given: SBX on every variable with those draws (the reference op); ``u=None``:
    the engine's draws for (seed, generation) -- per-pair Bernoulli(cfg.p_c), one u per variable --
    so the batch of all n/2 mating pairs reproduces the SBX half of :func:`vary_eval`."""
    P1, P2 = _pairs64(p1), _pairs64(p2)
    if P1.shape != P2.shape:
        raise ShapeError("p1 and p2 must have the same shape")
    npairs, d = P1.shape
    uu = None if u is None else _pairs64(u)
    if uu is not None and uu.shape != P1.shape:
        raise ShapeError("u must match the parents' shape")
    cfg = cfg or VariationConfig(eta_c=eta)
    C1, C2 = torch.empty_like(P1), torch.empty_like(P1)
    _lib.check(_lib.lib().mo_sbx_pairs(_lib.ptr(P1), _lib.ptr(P2), npairs, d, _lib.ptr(uu), float(cfg.eta_c),
                                       float(cfg.p_c), float(lo), float(hi), int(bool(clamp)), int(seed),
                                       int(generation), _lib.ptr(C1), _lib.ptr(C2), _lib.stream_ptr()),
               "mo_sbx_pairs")
    shape = as_cuda(p1, torch.float64).shape
    return C1.reshape(shape), C2.reshape(shape)


def polynomial_mutation(X, u=None, eta=20.0, lo=0.0, hi=1.0, flag=None, cfg=None, seed=0, generation=0):
    """Deb's bounded polynomial mutation of X, clamped to [lo, hi], FP64.  ``u``
    given: mutate where ``flag`` (everywhere when None) with those draws; ``u=None``: the engine's PM
    stream for (seed, generation) with rate cfg.p_m (1/d by default)."""
    Xt = _pairs64(X)
    n, d = Xt.shape
    uu = None if u is None else _pairs64(u)
    fl = None if flag is None else as_cuda(flag, torch.uint8).reshape(n, d)
    if uu is not None and uu.shape != Xt.shape:
        raise ShapeError("u must match X's shape")
    cfg = cfg or VariationConfig(eta_m=eta)
    p_m = 1.0 / d if cfg.p_m is None else cfg.p_m
    out = torch.empty_like(Xt)
    _lib.check(_lib.lib().mo_polynomial_mutation(_lib.ptr(Xt), n, d, _lib.ptr(uu), _lib.ptr(fl), float(cfg.eta_m),
                                                 float(p_m), float(lo), float(hi), int(seed), int(generation),
                                                 _lib.ptr(out), _lib.stream_ptr()), "mo_polynomial_mutation")
    return out.reshape(as_cuda(X, torch.float64).shape)


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
