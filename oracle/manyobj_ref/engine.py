"""Generational loop, Alg. 1 (oracle; TEST INFRASTRUCTURE ONLY).  SPEC.md:435-499.

``step`` = variation -> evaluation -> merge (parents first) ->
NDS with early exit at n -> split -> niching (batched | oracle back-end) ->
stable compaction in ascending merged index (A-9).  The RNG generation word
of step t is the number of steps already taken (``state.generation``).
"""
from dataclasses import dataclass, field, replace

import numpy as np

from paper_2504_06067_b200.errors import ConfigError
from . import dominance, niche, problems, refpoints
from . import variation as _variation
from . import rng as _rng


@dataclass(frozen=True)
class RunConfig:
    """SPEC.md:440-443."""
    problem: str = "DTLZ2"
    n: int = 92
    m: int = 3
    d: int = 12
    generations: int = 100
    seed: int = 0
    backend: str = "batched"
    variation: _variation.VariationConfig = _variation.VariationConfig()


@dataclass
class RunState:
    """SPEC.md:444-447."""
    generation: int
    X: np.ndarray
    F: np.ndarray
    ideal: np.ndarray
    zhat: np.ndarray
    Z: np.ndarray
    info: dict = field(default_factory=dict)


def validate(cfg):
    if cfg.n < cfg.m:
        raise ConfigError("n", "n must be >= m")
    if cfg.n % 2:
        raise ConfigError("n", "n must be even")
    if cfg.generations < 1:
        raise ConfigError("generations", "must be >= 1")
    if cfg.backend not in ("batched", "oracle"):
        raise ConfigError("backend", "batched | oracle")
    if cfg.problem not in problems.KINDS:
        raise ConfigError("problem", f"unknown {cfg.problem}")
    if cfg.d < cfg.m:
        raise ConfigError("d", "d must be >= m")


def evaluate(cfg, X):
    return problems.dtlz_eval(problems.ContinuousProblem(cfg.problem, cfg.m, cfg.d),
                              X).astype(np.float32)


def initial_population(n, d, seed):
    i = np.arange(n, dtype=np.int64)[:, None]
    v = np.arange(d, dtype=np.int64)[None, :]
    return _rng.uniform(seed, _rng.STREAM_INIT, 0, i, v)


def initialize(cfg):
    """SPEC.md:450-458."""
    validate(cfg)
    X = initial_population(cfg.n, cfg.d, cfg.seed)
    Z = refpoints.reference_points(cfg.m, cfg.n)
    F = evaluate(cfg, X)
    return RunState(0, X, F, F.min(axis=0), refpoints.unit_directions(Z), Z)


def survivor_selection(cfg, FR, ideal, zhat, generation, gen=None, loop="waterfill", nds_fn=None,
                       associate_fn=None, fast=False):
    """NDS + split + niching on merged objectives FR (2n x m FP32).

    ``nds_fn(FR, stop_at) -> ranks`` / ``associate_fn`` / ``fast``: the same stages from the C
    restatement (oracle/c, checked bit-for-bit against these numpy ones) for C2-C4-sized checks."""
    ranks = (nds_fn or (lambda F, stop_at: dominance.non_dominated_sort(F, stop_at=stop_at)))(FR, cfg.n)
    split = dominance.split_fronts(ranks, cfg.n)
    sel, info = niche.select(FR, ranks, split, ideal, zhat, cfg.seed, generation,
                             backend=cfg.backend, gen=gen, loop=loop, associate_fn=associate_fn, fast=fast)
    info["ranks"] = ranks
    return sel, info


def step(state, cfg, gen=None, offspring=None, loop="waterfill", **accel):
    """SPEC.md:459-467.  ``offspring=(O, FO)`` injects externally produced offspring; ``accel``:
    nds_fn / associate_fn / fast of :func:`survivor_selection`."""
    g = state.generation
    if offspring is None:
        O = _variation.vary(state.X, cfg.variation, cfg.seed, g)
        FO = evaluate(cfg, O)
    else:
        O, FO = (np.asarray(a, np.float32) for a in offspring)
    XR = np.concatenate([state.X, O])
    FR = np.concatenate([state.F, FO])
    sel, info = survivor_selection(cfg, FR, state.ideal, state.zhat, g, gen, loop, **accel)
    info["selected"] = sel
    return RunState(g + 1, XR[sel], FR[sel], info["ideal"], state.zhat, state.Z, info)


def run(cfg, gen=None):
    """per-generation records + final state."""
    state = initialize(cfg)
    history = []
    for _ in range(cfg.generations):
        state = step(state, cfg, gen=gen)
        history.append({"generation": state.generation, "l": state.info["l"],
                        "k": state.info["k"], "skipped": state.info["skipped"]})
    return history, state


def with_backend(cfg, backend):
    return replace(cfg, backend=backend)
