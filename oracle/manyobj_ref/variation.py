"""Mating pool, SBX, polynomial mutation (oracle; TEST INFRASTRUCTURE ONLY).

SPEC.md:238-308 with the pins of DESIGN.md:
* mating pool = permutation(n, stream MATING) split into consecutive pairs;
* per-pair Bernoulli(p_c) from Philox(q, PAIR_SLOT, g, SBX) (A-7), then one
  u per variable from Philox(q, v, g, SBX) word 0;
* PM flag u < p_m from Philox(i, v, g, PM) word 0, PM draw from word 1;
* clamp after each operator.
Arithmetic here is float64; the GPU computes in FP32 and is compared within
rtol 1e-5 (north star).
"""
from dataclasses import dataclass

import numpy as np

from paper_2504_06067_b200.errors import ParameterError
from . import rng as _rng


@dataclass(frozen=True)
class VariationConfig:
    """SPEC.md:243-246; defaults SPEC.md:293 (p_m=None -> 1/d)."""
    eta_c: float = 20.0
    eta_m: float = 20.0
    p_c: float = 1.0
    p_m: float = None


def mating_pool(n, seed, generation):
    """(n/2, 2) parent index pairs."""
    if n % 2:
        raise ParameterError("mating pool needs even n")
    perm = _rng.permutation(n, seed, generation, _rng.STREAM_MATING)
    return perm.reshape(-1, 2)


def sbx_beta(u, eta):
    u = np.asarray(u, dtype=np.float64)
    e = 1.0 / (eta + 1.0)
    lo = np.power(2.0 * u, e)
    with np.errstate(divide="ignore"):
        hi = np.power(1.0 / (2.0 * (1.0 - u)), e)
    return np.where(u <= 0.5, lo, hi)


def sbx_pair(p1, p2, u, eta, lo=0.0, hi=1.0, clamp=True):
    """Children of one pair given per-variable u."""
    b = sbx_beta(u, eta)
    c1 = 0.5 * ((1.0 + b) * p1 + (1.0 - b) * p2)
    c2 = 0.5 * ((1.0 - b) * p1 + (1.0 + b) * p2)
    if clamp:
        c1 = np.clip(c1, lo, hi)
        c2 = np.clip(c2, lo, hi)
    return c1, c2


def pm_delta(x, u, eta, lo=0.0, hi=1.0):
    """Deb's bounded polynomial mutation of x with draw u."""
    x = np.asarray(x, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    span = hi - lo
    d1 = (x - lo) / span
    d2 = (hi - x) / span
    mp = 1.0 / (eta + 1.0)
    v_lo = 2.0 * u + (1.0 - 2.0 * u) * np.power(1.0 - d1, eta + 1.0)
    v_hi = 2.0 * (1.0 - u) + 2.0 * (u - 0.5) * np.power(1.0 - d2, eta + 1.0)
    dq = np.where(u < 0.5, np.power(v_lo, mp) - 1.0, 1.0 - np.power(v_hi, mp))
    return x + dq * span


def vary(X, cfg, seed, generation, lo=0.0, hi=1.0):
    """n offspring of parents X (n x d) for generation ``generation``."""
    X = np.asarray(X, dtype=np.float32)
    n, d = X.shape
    p_m = np.float32(1.0 / d if cfg.p_m is None else cfg.p_m)
    p_c = np.float32(cfg.p_c)
    pairs = mating_pool(n, seed, generation)
    q = np.arange(n // 2, dtype=np.int64)
    v = np.arange(d, dtype=np.int64)
    u_pair = _rng.uniform(seed, _rng.STREAM_SBX, generation, q, _rng.PAIR_SLOT)
    u_var = _rng.uniform(seed, _rng.STREAM_SBX, generation, q[:, None], v[None, :])
    p1 = X[pairs[:, 0]].astype(np.float64)
    p2 = X[pairs[:, 1]].astype(np.float64)
    c1, c2 = sbx_pair(p1, p2, u_var, cfg.eta_c, lo, hi)
    cross = (u_pair < p_c)[:, None]
    c1 = np.where(cross, c1, p1)
    c2 = np.where(cross, c2, p2)
    O = np.empty((n, d), dtype=np.float64)
    O[0::2] = c1
    O[1::2] = c2
    i = np.arange(n, dtype=np.int64)
    draws = _rng.philox4x32(i[:, None], v[None, :], generation, _rng.STREAM_PM, seed)
    flag = _rng.u01(draws[0]) < p_m
    u_pm = _rng.u01(draws[1])
    # the GPU feeds PM the FP32-rounded SBX child; do the same before mutating
    O32 = O.astype(np.float32).astype(np.float64)
    mutated = np.clip(pm_delta(O32, u_pm, cfg.eta_m, lo, hi), lo, hi)
    O = np.where(flag, mutated, O32)
    return O.astype(np.float32)
