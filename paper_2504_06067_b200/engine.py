"""The generational loop of NSGA-III (Alg. 1) on one B200 -- the drop-in ``engine``.

Reference interface: engine.RunConfig / RunState / initialize / step / run
(SPEC.md:435-499).  One generation is one ``mo_step`` C-ABI call (variation +
evaluation, dominance bit-matrix + peeling, normalisation + association +
niching + survivor compaction), entirely stream-ordered on the device.

State lives in two ping-pong merged buffers (2n rows each): parents occupy
rows [0, n) of the current buffer, offspring are written to rows [n, 2n),
survivors are compacted into rows [0, n) of the other buffer.  No copies, no
host round trip per generation.  With ``graph=True`` each generation is one
CUDA-graph replay (one graph per buffer parity); the generation counter lives
in device memory so the same two graphs are replayed generation after
generation.

Only the ``batched`` back-end exists here: the Alg. 1 one-at-a-time oracle
 is CPU test infrastructure (oracle/manyobj_ref) and asking
for it raises ConfigError rather than falling back to the CPU.
"""
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, problems, refpoints
from .errors import ConfigError
from .variation import VariationConfig, init_population


@dataclass(frozen=True)
class RunConfig:
    """problem, n (even, >= m), m, d, generations, seed, backend, variation."""
    problem: str = "DTLZ2"
    n: int = 92
    m: int = 3
    d: int = 12
    generations: int = 100
    seed: int = 0
    backend: str = "batched"
    variation: VariationConfig = VariationConfig()
    reference_points: tuple = None   # (H_outer, H_inner); None = choose_divisions(m, n)


def validate(cfg):
    if cfg.problem not in problems.KINDS:
        raise ConfigError("problem", f"unknown problem {cfg.problem!r}")
    if cfg.m < 2:
        raise ConfigError("m", "need m >= 2")
    if cfg.n < cfg.m:
        raise ConfigError("n", "n must be >= m")
    if cfg.n % 2:
        raise ConfigError("n", "n must be even")
    if cfg.d < cfg.m:
        raise ConfigError("d", "d must be >= m")
    if cfg.generations < 1:
        raise ConfigError("generations", "must be >= 1")
    if cfg.m > 16:
        raise ConfigError("m", "the association kernels are instantiated for m <= 16")
    if cfg.backend != "batched":
        raise ConfigError("backend", "the GPU engine implements the batched back-end only; the Alg. 1 "
                                     "oracle back-end is CPU test infrastructure (oracle/manyobj_ref)")


def build_reference_set(cfg):
    if cfg.reference_points is None:
        Z = refpoints.reference_points(cfg.m, cfg.n)
    else:
        Ho, Hi = cfg.reference_points
        Z = refpoints.two_layer(cfg.m, Ho, Hi) if Hi else refpoints.das_dennis(cfg.m, Ho)
    return Z, refpoints.unit_directions(Z)


class Engine:
    """Device-resident NSGA-III run: buffers, workspace and (optionally) a CUDA graph."""

    def __init__(self, cfg, graph=False, device=None):
        validate(cfg)
        self.cfg = cfg
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n, m, d = cfg.n, cfg.m, cfg.d
        self.problem = problems.ContinuousProblem(cfg.problem, m, d)
        self.Z, zh = build_reference_set(cfg)
        self.w = zh.shape[0]
        with torch.cuda.device(self.dev):
            L = _lib.lib()
            self.zhat = torch.from_numpy(zh).to(self.dev)
            self.XR = [torch.empty((2 * n, d), dtype=torch.float32, device=self.dev) for _ in range(2)]
            self.FR = [torch.empty((2 * n, m), dtype=torch.float32, device=self.dev) for _ in range(2)]
            self.ranks = torch.empty(2 * n, dtype=torch.int32, device=self.dev)
            self.info = torch.zeros(_lib.INFO_COUNT, dtype=torch.int32, device=self.dev)
            self.gen_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self.ws = _lib.workspace_step(n, m, d, self.w, self.dev)
            X0 = init_population(n, d, cfg.seed)
            self.XR[0][:n].copy_(X0)
            self.FR[0][:n].copy_(problems.dtlz_eval(self.problem, X0))
            self.ideal = self.FR[0][:n].amin(dim=0).contiguous()   # running ideal starts at min(F_0)
            del L
        self.cur = 0
        self.generation = 0
        self._args = [self._make_args(0), self._make_args(1)]
        self._graph = None
        if graph:
            self.capture()

    # ------------------------------------------------------------ C-ABI args
    def _make_args(self, cur, use_dev_gen=False):
        cfg = self.cfg
        n = cfg.n
        a = _lib.StepArgs()
        a.problem = self.problem.id
        a.m, a.d, a.n, a.w = cfg.m, cfg.d, n, self.w
        a.seed = int(cfg.seed)
        a.generation = 0
        a.var = cfg.variation.c_struct()
        a.zhat = self.zhat.data_ptr()
        a.XR = self.XR[cur].data_ptr()
        a.FR = self.FR[cur].data_ptr()
        a.X_next = self.XR[1 - cur].data_ptr()
        a.F_next = self.FR[1 - cur].data_ptr()
        a.ideal = self.ideal.data_ptr()
        a.ranks = self.ranks.data_ptr()
        a.info = self.info.data_ptr()
        a.workspace = self.ws.data_ptr()
        a.workspace_bytes = self.ws.numel()
        a.generation_dev = self.gen_dev.data_ptr() if use_dev_gen else None
        return a

    def _launch(self, cur, generation, phases=_lib.PHASE_ALL, use_dev_gen=False):
        a = self._make_args(cur, use_dev_gen) if use_dev_gen else self._args[cur]
        a.generation = int(generation) & 0xFFFFFFFF
        _lib.check(_lib.lib().mo_step_phases(a, phases, _lib.stream_ptr()), "mo_step")

    # ------------------------------------------------------------- stepping
    def step(self, profile=None):
        """Advance one generation (eager launch).  ``profile``: dict receiving per-phase ms."""
        if profile is None:
            self._launch(self.cur, self.generation)
        else:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            self._launch(self.cur, self.generation, _lib.PHASE_VARY)
            ev[1].record()
            self._launch(self.cur, self.generation, _lib.PHASE_SORT)
            ev[2].record()
            self._launch(self.cur, self.generation, _lib.PHASE_NICHE)
            ev[3].record()
            ev[3].synchronize()
            for name, a, b in (("t_variation", 0, 1), ("t_sort", 1, 2), ("t_niche", 2, 3)):
                profile[name] = profile.get(name, 0.0) + ev[a].elapsed_time(ev[b]) / 1e3
            profile["t_eval"] = profile.get("t_eval", 0.0)   # fused into t_variation (k_vary_eval)
        self.cur ^= 1
        self.generation += 1

    def capture(self):
        """Capture one generation per buffer parity (A->B and B->A) as two CUDA graphs."""
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        graphs = []
        for cur in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self._launch(cur, 0, use_dev_gen=True)
            graphs.append(g)
        torch.cuda.current_stream().wait_stream(s)
        self._graph = graphs

    def replay_one(self):
        """Advance one generation by replaying the captured graph of the current parity."""
        if self._graph is None:
            raise RuntimeError("no graph captured")
        self._graph[self.cur].replay()
        self.cur ^= 1
        self.generation += 1

    def replay(self, generations=1):
        """Advance ``generations`` generations with graph replays (device generation counter)."""
        if self._graph is None:
            raise RuntimeError("no graph captured")
        self.gen_dev.fill_(self.generation)
        for _ in range(generations):
            self.replay_one()

    # --------------------------------------------------------------- views
    @property
    def X(self):
        return self.XR[self.cur][: self.cfg.n]

    @property
    def F(self):
        return self.FR[self.cur][: self.cfg.n]

    TRACE_SLOTS = {
        "presort.sum": (0, 1), "presort.hist": (1, 2), "presort.scan": (2, 3), "presort.scatter": (3, 4),
        "presort.bounds": (4, 5),
        "peel.prologue": (8, 9), "peel.fronts": (9, 10),
        "prep.phase0": (16, 17), "prep.extremes": (17, 18), "prep.solve": (18, 19),
        "select.nearest_keys": (24, 25), "select.nearest": (25, 26), "select.level": (26, 27),
        "select.marked": (27, 28), "select.take": (28, 29), "select.cache": (29, 30), "select.topk": (30, 31),
        "select.compact": (31, 35), "select.ranks": (35, 36), "select.total": (24, 36),
    }

    def trace(self):
        """Phase durations (us) inside the persistent kernels of the last step (globaltimer)."""
        off = int(_lib.lib().mo_trace_offset(self.cfg.n, self.cfg.m, self.w))
        t = self.ws[off: off + 64 * 8].view(torch.int64).cpu().tolist()
        out = {}
        for name, (a, b) in self.TRACE_SLOTS.items():
            if t[a] and t[b] and t[b] >= t[a]:
                out[name] = (t[b] - t[a]) / 1e3
        return out

    def info_dict(self):
        h = self.info.cpu().tolist()
        return {k.lower(): h[v] for k, v in _lib.INFO.items()}


@dataclass
class RunState:
    """SPEC.md:444-447.  X/F are views into the engine's ping-pong buffers
    (valid until the next-but-one step; ``.clone()`` them to keep)."""
    generation: int
    X: torch.Tensor
    F: torch.Tensor
    ideal: torch.Tensor
    engine: Engine = field(repr=False)
    timings: dict = field(default_factory=dict)

    @property
    def Z(self):
        return self.engine.Z


def _state(engine, timings):
    return RunState(engine.generation, engine.X, engine.F, engine.ideal, engine, timings)


def initialize(cfg, graph=False):
    """uniform population in bounds, evaluated; generation 0."""
    eng = Engine(cfg, graph=graph)
    return _state(eng, {})


def step(state, cfg=None, profile=False):
    """one generation; returns the advanced state."""
    eng = state.engine
    if cfg is not None and cfg != eng.cfg:
        raise ConfigError("cfg", "state was initialised with a different RunConfig")
    timings = dict(state.timings)
    eng.step(profile=timings if profile else None)
    return _state(eng, timings)


def run(cfg, record=True, profile=False, graph=False):
    """history of per-generation records + final state."""
    state = initialize(cfg, graph=graph and not record and not profile)
    eng = state.engine
    history = []
    g = cfg.generations
    if eng._graph is not None:
        eng.replay(g)
        return history, _state(eng, {})
    for _ in range(g):
        state = step(state, profile=profile)
        if record:
            info = eng.info_dict()
            history.append({"generation": state.generation, "l": info["l"], "k": info["k"],
                            "fronts": info["nfronts"], "skipped": info["skipped"],
                            "survivors": info["survivors"]})
    return history, state


__all__ = ["RunConfig", "RunState", "Engine", "initialize", "step", "run", "validate", "build_reference_set"]
