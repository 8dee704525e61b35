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

Sort modes (``sort=``): "bits" keeps the R x R dominance bit-matrix in HBM
and runs a generation as one ``mo_step`` (graph-capturable); "stream" never
stores it (O(R) memory) and peels front by front from the host through
``mo_sort_stream_*`` -- the path for populations whose bit-matrix exceeds
HBM (C4: R = 2M) and for sharding.  "auto" picks bits when it fits.

Sharding (``group=`` a torch.distributed process group, one process per
GPU): the streamed sort's dominated rows are dealt to the shards in
256-row position blocks and the per-front masks all-gathered; the
association splits the reference points and max-reduces the packed
(key, position) words; everything else is replicated, so every shard holds
the same survivors, bit-identical to one GPU.  A
generation is written as a generator that yields its collectives, so the
same code runs under NCCL, gloo, or an in-process emulation of G shards on
one device (``LocalShards``, used by the tests).

Only the ``batched`` back-end exists here: the Alg. 1 one-at-a-time oracle
 is CPU test infrastructure (oracle/manyobj_ref) and asking
for it raises ConfigError rather than falling back to the CPU.
"""
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, problems, refpoints
from .errors import ConfigError, ShapeError, raise_for_status
from .variation import VariationConfig, init_population


MAX_M = 512   # include/manyobj_b200.h MO_MAX_M: m > 16 runs the runtime-m ("wide") kernels


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
    if cfg.m > MAX_M:
        raise ConfigError("m", f"m <= {MAX_M} (PAPER.md Appendix D's largest objective count)")
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

    def __init__(self, cfg, graph=False, device=None, sort="auto", group=None, shard=None, poll=4, prune="auto",
                 host_fronts=None, prune_r=0, debug=False):
        """``debug``: after every eager step, recompute the niche bookkeeping from scratch
        (niche.check_bookkeeping) and keep the niche trace records in
        ``self.niche_trace``; raises RuntimeError on the first inconsistency.  Costs host syncs."""
        validate(cfg)
        self.cfg = cfg
        self.debug = bool(debug)
        self.niche_trace = []
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n, m, d = cfg.n, cfg.m, cfg.d
        self.problem = problems.ContinuousProblem(cfg.problem, m, d)
        self.Z, zh = build_reference_set(cfg)
        self.w = zh.shape[0]
        self.group = group
        if shard is None:
            shard = (0, 1)
            if group is not None:
                import torch.distributed as dist
                shard = (dist.get_rank(group), dist.get_world_size(group))
        self.shard_rank, self.shard_count = int(shard[0]), int(shard[1])
        if not (0 <= self.shard_rank < self.shard_count):
            raise ConfigError("shard", f"bad shard {shard}")
        self.sort_mode = self._choose_sort(sort)
        self.poll = max(1, int(poll))
        self.prune_r = int(prune_r)          # lattice box radius (0 = the library default for m)
        # streamed sort, one shard: the front loop either runs on the device inside mo_step (one
        # cooperative launch, graph-capturable; ~30 us per front) or front by front from the host
        # (full-occupancy sweep launches, ~50 us per front; faster when the sweeps dominate, e.g. C4).
        # host_fronts=None (auto, eager): host-driven while the previous generation had <= 300 fronts,
        # device-side beyond (profiles/r01_sort_modes.jsonl: DTLZ4 m=3 has thousands).  Sharded runs
        # are always host-driven: the collectives sit between the fronts.
        self._auto_fronts = host_fronts is None and not graph
        if host_fronts is None:
            host_fronts = not graph
        self.host_fronts = self.sort_mode == _lib.SORT_STREAM and (self.shard_count > 1 or bool(host_fronts))
        self._fronts_hint = 0
        if graph and self.host_fronts:
            raise ConfigError("graph", "CUDA-graph replay needs the device-side front loop (one shard)")
        with torch.cuda.device(self.dev):
            L = _lib.lib()
            self.zhat = torch.from_numpy(zh).to(self.dev)
            self.lattice, self.lattice_H = self._lattice_table(prune)   # (z, index, pos) or None
            # bf16 hi/lo MMA fragments of the unit directions (tensor-core filter of the full-scan
            # association; static, packed once)
            # and the FP16 UMMA tiles of the tcgen05 filter, preferred by the library when both are set)
            self.zfrag = self.zumma = None
            if self.lattice is None and 2 <= m <= 16 and self.shard_count == 1:
                self.zfrag = torch.empty(int(L.mo_pack_refs_bytes(self.w)), dtype=torch.uint8, device=self.dev)
                self.zumma = torch.empty(int(L.mo_pack_refs_f16_bytes(self.w, m)), dtype=torch.uint8, device=self.dev)
                order = torch.from_numpy(np.random.default_rng(0x5EED).permutation(self.w).astype(np.int32))
                order = order.to(self.dev)
                _lib.check(L.mo_pack_refs_bf16(self.zhat.data_ptr(), self.w, m, order.data_ptr(),
                                               self.zfrag.data_ptr(), _lib.stream_ptr()), "mo_pack_refs_bf16")
                _lib.check(L.mo_pack_refs_f16(self.zhat.data_ptr(), self.w, m, order.data_ptr(),
                                              self.zumma.data_ptr(), _lib.stream_ptr()), "mo_pack_refs_f16")
                torch.cuda.current_stream(self.dev).synchronize()   # `order` is freed on return
            self.XR = [torch.empty((2 * n, d), dtype=torch.float32, device=self.dev) for _ in range(2)]
            self.FR = [torch.empty((2 * n, m), dtype=torch.float32, device=self.dev) for _ in range(2)]
            self.ranks = torch.empty(2 * n, dtype=torch.int32, device=self.dev)
            self.info = torch.zeros(_lib.INFO_COUNT, dtype=torch.int32, device=self.dev)
            self.gen_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
            nbytes = _lib.workspace_bytes_ex(n, m, d, self.w, self.sort_mode, self.shard_count)
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
            _lib.check(L.mo_workspace_init(self.ws.data_ptr(), nbytes, _lib.stream_ptr()), "mo_workspace_init")
            if self.sort_mode == _lib.SORT_STREAM:
                lo, words, fo, ao = _lib.stream_offsets(n, m, self.w, self.sort_mode, self.shard_count)
                self.mask_local = self.ws[lo: lo + 4 * words].view(torch.int32)
                self.mask_full = self.ws[fo: fo + 4 * words * self.shard_count].view(torch.int32)
                self.akey = self.ws[ao: ao + 8 * 2 * n].view(torch.int64)
            X0 = init_population(n, d, cfg.seed)
            self.XR[0][:n].copy_(X0)
            self.FR[0][:n].copy_(problems.dtlz_eval(self.problem, X0))
            self.ideal = self.FR[0][:n].amin(dim=0).contiguous()   # running ideal starts at min(F_0)
            del L
        self.cur = 0
        self.generation = 0
        self._gen_dev_synced = True      # gen_dev == self.generation (graph replays read it)
        # sticky device status (info[ERROR_FIRST]) copied to pinned memory after every eager step and
        # raised lazily by the next step / check_errors() -- no host sync per generation
        self._err_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self._err_event = None
        self._args = [self._make_args(0), self._make_args(1)]
        self._graph = None
        if graph:
            self.capture()

    def _lattice_table(self, prune):
        """Dense (k_0..k_{m-2}) -> reference index table for the exact lattice-pruned association
        (single-layer Das-Dennis, m <= 4).  prune: "auto" (when it pays), True (whenever legal), False."""
        cfg, m, w = self.cfg, self.cfg.m, self.w
        Ho, Hi = cfg.reference_points if cfg.reference_points is not None else refpoints.choose_divisions(m, cfg.n)
        legal = Hi == 0 and 2 <= m <= 5 and (Ho + 1) ** (m - 1) <= (1 << 26)
        if prune is False or not legal:
            if prune is True and not legal:
                raise ConfigError("prune", "lattice pruning needs a single-layer Das-Dennis set and m <= 5")
            return None, 0
        r = self.prune_r or (6 if m <= 3 else (3 if m == 4 else 1))   # default_lattice_r (mo_capi.cu)
        # a box point costs several full-scan points (decode + gathered loads); measured: C2 (m=5, w=8855,
        # r=2) 185 -> 167 us niche phase, m=5 N=100k 6.2 -> 0.54 ms (scripts/assoc_probe.py)
        if prune == "auto" and 8 * (2 * r - 1) ** (m - 1) >= w:     # box of (2r-1)^(m-1) points
            return None, 0
        k = np.rint(np.asarray(self.Z, np.float64) * Ho).astype(np.int64)
        idx = np.zeros(w, np.int64)
        for i in range(m - 1):
            idx = idx * (Ho + 1) + k[:, i]
        size = (Ho + 1) ** (m - 1)
        zl = np.zeros((size, m), np.float32)
        zl[idx] = self.zhat.cpu().numpy()              # the same FP32 directions the full scan reads
        dev = lambda x: torch.from_numpy(x).to(self.dev)
        return (dev(zl), dev(idx.astype(np.int32)), torch.zeros(size, dtype=torch.int32, device=self.dev)), Ho

    def _choose_sort(self, sort):
        if sort not in ("auto", "bits", "stream"):
            raise ConfigError("sort", f"unknown sort mode {sort!r}")
        if sort == "bits" and self.shard_count > 1:
            raise ConfigError("sort", "the sharded sort is the streamed one")
        if sort == "auto":
            R = 2 * self.cfg.n
            bits = R * ((R + 255) // 256 * 8) * 4
            budget = 0.5 * torch.cuda.get_device_properties(self.dev).total_memory
            # measured crossovers: the boxed streamed sort overtakes the bit-matrix at n ~ 100k for m = 3
            # (profiles/r01_sort_modes.jsonl); for m >= 4 the rank-mask bit-matrix sort (round 2) is
            # faster wherever the matrix fits (C3: 9.9 ms per generation vs 25 ms streamed)
            n, m = self.cfg.n, self.cfg.m
            boxed_wins = m <= 3 and n >= 100_000
            sort = "bits" if self.shard_count == 1 and bits <= budget and not boxed_wins else "stream"
            if sort == "stream" and m > 16:
                raise ConfigError("m", "the streamed sort runs m <= 16; this population's bit-matrix does "
                                       "not fit the device")
        if sort == "stream" and self.cfg.m > 16:
            raise ConfigError("sort", "the streamed / sharded sort runs m <= 16")
        return _lib.SORT_BITS if sort == "bits" else _lib.SORT_STREAM

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
        a.sort_mode = self.sort_mode
        a.shard_rank, a.shard_count = self.shard_rank, self.shard_count
        if self.lattice is not None:
            a.lattice_z, a.lattice_index, a.lattice_pos = (t.data_ptr() for t in self.lattice)
        a.lattice_H = self.lattice_H
        a.lattice_r = self.prune_r
        a.zhat_frag = self.zfrag.data_ptr() if self.zfrag is not None else None
        a.zhat_umma = self.zumma.data_ptr() if self.zumma is not None else None
        Ho, Hi = (cfg.reference_points if cfg.reference_points is not None
                  else refpoints.choose_divisions(cfg.m, cfg.n))
        a.ref_H_outer, a.ref_H_inner = int(Ho), int(Hi)
        return a

    def _launch(self, cur, generation, phases=_lib.PHASE_ALL, use_dev_gen=False):
        a = self._make_args(cur, use_dev_gen) if use_dev_gen else self._args[cur]
        a.generation = int(generation) & 0xFFFFFFFF
        _lib.check(_lib.lib().mo_step_phases(a, phases, _lib.stream_ptr()), "mo_step")

    # ------------------------------------------------------------- stepping
    def step(self, profile=None):
        """Advance one generation (eager launch).  ``profile``: dict receiving per-phase seconds.

        A device-side failure of an earlier generation (e.g. InfeasibleSplitError) is raised here, at
        the latest one step late, or by :meth:`check_errors`."""
        self.check_errors(block=False)
        self._step_dispatch(profile)
        self._gen_dev_synced = False
        self._post_error_copy()
        if self.debug:
            from . import niche
            self.check_errors(block=True)
            self.niche_trace.append(niche.trace(self))
            bad = [k for k, ok in niche.check_bookkeeping(self).items() if not ok]
            if bad:
                raise RuntimeError(f"niche bookkeeping mismatch at generation {self.generation - 1}: {bad}")

    # ------------------------------------------------------------ snapshots
    def snapshot(self):
        """Run-state snapshot: the population, its objectives, the running ideal,
        the generation counter and the configuration -- everything a generation depends on (the
        keyed RNG streams are functions of (seed, generation)), so a restored engine continues
        bit-identically.  Host numpy arrays + plain values."""
        import dataclasses
        self.check_errors(block=True)
        cfg = dataclasses.asdict(self.cfg)
        return {"format": "manyobj_b200.snapshot/1", "generation": int(self.generation), "config": cfg,
                "X": self.X.cpu().numpy().copy(), "F": self.F.cpu().numpy().copy(),
                "ideal": self.ideal.cpu().numpy().copy()}

    def restore(self, snap):
        """Load a :meth:`snapshot` of a run with the same configuration into this engine."""
        import dataclasses
        if snap.get("format") != "manyobj_b200.snapshot/1":
            raise ConfigError("snapshot", "unknown snapshot format")
        import json

        def canon(c):   # JSON form: tuples and lists compare equal
            c = json.loads(json.dumps(c, default=_json_default))
            c.pop("generations", None)
            return c
        if canon(dataclasses.asdict(self.cfg)) != canon(dict(snap["config"])):
            raise ConfigError("snapshot", "snapshot of a different RunConfig")
        n, m, d = self.cfg.n, self.cfg.m, self.cfg.d
        X = torch.as_tensor(np.asarray(snap["X"], np.float32))
        F = torch.as_tensor(np.asarray(snap["F"], np.float32))
        if X.shape != (n, d) or F.shape != (n, m):
            raise ShapeError(f"snapshot population {tuple(X.shape)} / {tuple(F.shape)}")
        self.XR[self.cur][:n].copy_(X)
        self.FR[self.cur][:n].copy_(F)
        self.ideal.copy_(torch.as_tensor(np.asarray(snap["ideal"], np.float32)))
        self.generation = int(snap["generation"])
        self._gen_dev_synced = False
        torch.cuda.synchronize(self.dev)

    def _post_error_copy(self):
        self._err_host.copy_(self.info[_lib.INFO["ERROR_FIRST"]: _lib.INFO["ERROR_FIRST"] + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._err_event = ev

    def check_errors(self, block=True):
        """Raise the reference exception of the first device-side status since the last check
        (errors.STATUS_TO_ERROR).  block=False only looks at copies that already landed."""
        if block:
            torch.cuda.current_stream(self.dev).synchronize()
            code = int(self.info[_lib.INFO["ERROR_FIRST"]].item())
        else:
            if self._err_event is None or not self._err_event.query():
                return
            code = int(self._err_host[0])
        self._err_event = None
        if code:
            self.info[_lib.INFO["ERROR_FIRST"]] = 0
            self._err_host.zero_()
            raise_for_status(code, f"engine generation <= {self.generation}")

    def _step_dispatch(self, profile=None):
        device_fronts = (self._auto_fronts and self.shard_count == 1 and self.sort_mode == _lib.SORT_STREAM
                         and self._fronts_hint > 300)
        if self.host_fronts and not device_fronts:
            for req in self.step_gen(profile):
                run_collective(req, self.group)
            return
        if device_fronts:
            self._step_device(profile)
            self._fronts_hint = int(self.info[_lib.INFO["NFRONTS"]].item())
            return
        self._step_device(profile)

    def _step_device(self, profile=None):
        """One generation through mo_step / mo_step_phases (device-side front loop when streamed)."""
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

    def _lib(self):
        return _lib.lib()

    def _stream(self):
        return _lib.stream_ptr()

    def step_gen(self, profile=None):
        """One streamed/sharded generation; yields its collectives (see run_collective).
        The host logic here (order of the collectives, lazy split polling, lockstep exit) is shared by
        NCCL runs, the in-process LocalShards emulation and the gloo CPU tests."""
        L, s = self._lib(), self._stream()
        a = self._args[self.cur]
        a.generation = int(self.generation) & 0xFFFFFFFF
        sharded = self.shard_count > 1
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if profile is not None else None
        if ev:
            ev[0].record()
        _lib.check(L.mo_step_phases(a, _lib.PHASE_VARY, s), "mo_step_phases(VARY)")
        if ev:
            ev[1].record()
        _lib.check(L.mo_sort_stream_begin(a, s), "mo_sort_stream_begin")
        k = 0
        while True:
            if sharded:
                yield ("all_gather", self.mask_local, self.mask_full)
            _lib.check(L.mo_sort_stream_front(a, k, s), "mo_sort_stream_front")
            k += 1
            if k % self.poll == 0 or k == 1:
                nf = int(self.info[_lib.INFO["NFRONTS"]].item())
                if nf > 0:   # identical on every shard
                    self._fronts_hint = nf
                    break
        _lib.check(L.mo_sort_stream_end(a, s), "mo_sort_stream_end")
        if ev:
            ev[2].record()
        if sharded:
            _lib.check(L.mo_niche_phases(a, _lib.NICHE_PREP | _lib.NICHE_ASSOC, s), "mo_niche_phases")
            yield ("all_max_u64", self.akey)
            _lib.check(L.mo_niche_phases(a, _lib.NICHE_FINISH, s), "mo_niche_phases")
        else:
            _lib.check(L.mo_step_phases(a, _lib.PHASE_NICHE, s), "mo_step_phases(NICHE)")
        if ev:
            ev[3].record()
            ev[3].synchronize()
            for name, i, j in (("t_variation", 0, 1), ("t_sort", 1, 2), ("t_niche", 2, 3)):
                profile[name] = profile.get(name, 0.0) + ev[i].elapsed_time(ev[j]) / 1e3
            profile["t_eval"] = profile.get("t_eval", 0.0)
            profile["fronts_issued"] = k
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
        if not self._gen_dev_synced:      # eager steps advanced the host counter only
            self.gen_dev.fill_(self.generation)
            self._gen_dev_synced = True
        self._graph[self.cur].replay()
        self.cur ^= 1
        self.generation += 1

    def replay(self, generations=1, check=True):
        """Advance ``generations`` generations with graph replays (device generation counter);
        device-side errors are raised at the end (check=True: one host sync)."""
        if self._graph is None:
            raise RuntimeError("no graph captured")
        self.gen_dev.fill_(self.generation)
        self._gen_dev_synced = True
        for _ in range(generations):
            self.replay_one()
        if check:
            self.check_errors(block=True)

    # --------------------------------------------------------------- views
    @property
    def X(self):
        return self.XR[self.cur][: self.cfg.n]

    @property
    def F(self):
        return self.FR[self.cur][: self.cfg.n]

    TRACE_SLOTS = {
        "vary.parents": (40, 41), "vary.sbx_pm": (41, 42), "vary.g": (42, 43), "vary.objectives": (43, 44),
        "vary.prologue": (46, 45), "vary.prologue_end_to_vary_end": (45, 44),
        "presort.sum": (0, 1), "presort.hist": (1, 2), "presort.scan": (2, 3), "presort.scatter": (3, 4),
        "presort.bounds": (4, 5),
        "peel.prologue": (8, 9), "peel.fronts": (9, 10),
        "prep.phase0": (16, 17), "prep.extremes": (17, 18), "prep.solve": (18, 19),
        "prep.solve_loads": (18, 20), "prep.solve_gauss": (20, 21), "prep.solve_icpt": (21, 19),
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
        # (the sticky ERROR_FIRST slot is left for check_errors to raise)
        return {k.lower(): h[v] for k, v in _lib.INFO.items()}


_SIGN64 = -(1 << 63)


def run_collective(req, group):
    """Execute one collective request of Engine.step_gen over torch.distributed.

    NCCL moves the device buffers directly (NVLink).  Under gloo with device
    buffers (several processes sharing one GPU in the tests) the bytes are
    staged through host memory; the collective itself is the same."""
    import torch.distributed as dist
    kind = req[0]
    staged = req[1].is_cuda and dist.get_backend(group) == "gloo"
    if kind == "all_gather":
        src, dst = req[1], req[2]
        if staged:
            host = dst.cpu()
            dist.all_gather_into_tensor(host, src.cpu(), group=group)
            dst.copy_(host)
        else:
            dist.all_gather_into_tensor(dst, src, group=group)
    elif kind == "all_max_u64":
        # packed (ord(t), ~position) keys are unsigned: flip the sign bit so the signed max agrees
        t = req[1]
        t.bitwise_xor_(_SIGN64)
        if staged:
            host = t.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.MAX, group=group)
            t.copy_(host)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        t.bitwise_xor_(_SIGN64)
    else:
        raise ValueError(kind)


class LocalShards:
    """G shards of one run emulated in one process on one device: every shard
    is a full Engine; collectives are performed by concatenation / elementwise
    max across the shards' buffers.  Results must be bit-identical to G
    processes over NCCL (the kernels only see their shard index)."""

    def __init__(self, cfg, shards, device=None, poll=4, prune="auto"):
        self.engines = [Engine(cfg, device=device, sort="stream", shard=(g, shards), poll=poll, prune=prune,
                               host_fronts=True) for g in range(shards)]

    def step(self):
        gens = [e.step_gen() for e in self.engines]
        while True:
            reqs = []
            for g in gens:
                try:
                    reqs.append(next(g))
                except StopIteration:
                    reqs.append(None)
            if all(r is None for r in reqs):
                return
            if any(r is None for r in reqs) or len({r[0] for r in reqs}) != 1:
                raise RuntimeError("shards diverged: " + repr([r and r[0] for r in reqs]))
            if reqs[0][0] == "all_gather":
                full = torch.cat([r[1] for r in reqs])
                for r in reqs:
                    r[2].copy_(full)
            else:
                ts = [r[1] ^ _SIGN64 for r in reqs]
                mx = ts[0]
                for t in ts[1:]:
                    mx = torch.maximum(mx, t)
                mx ^= _SIGN64
                for r in reqs:
                    r[1].copy_(mx)


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


def initialize(cfg, graph=False, **engine_kw):
    """uniform population in bounds, evaluated; generation 0.
    ``engine_kw``: Engine options (sort=, group=, device=)."""
    eng = Engine(cfg, graph=graph, **engine_kw)
    return _state(eng, {})


def step(state, cfg=None, profile=False):
    """one generation; returns the advanced state."""
    eng = state.engine
    if cfg is not None and cfg != eng.cfg:
        raise ConfigError("cfg", "state was initialised with a different RunConfig")
    timings = dict(state.timings)
    eng.step(profile=timings if profile else None)
    return _state(eng, timings)


def run(cfg, record=True, profile=False, graph=False, **engine_kw):
    """history of per-generation records + final state."""
    state = initialize(cfg, graph=graph and not record and not profile, **engine_kw)
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
    eng.check_errors(block=True)
    return history, state


def save_state(state, path):
    """Write a run-state snapshot (Engine.snapshot) to ``path`` (numpy .npz; SPEC.md:492's optional binary
    snapshot of the population)."""
    import json
    snap = state.engine.snapshot() if isinstance(state, RunState) else state.snapshot()
    meta = {"format": snap["format"], "generation": snap["generation"], "config": snap["config"]}
    np.savez(path, X=snap["X"], F=snap["F"], ideal=snap["ideal"],
             meta=np.frombuffer(json.dumps(meta, default=_json_default).encode(), dtype=np.uint8))


def _json_default(o):
    import dataclasses
    if dataclasses.is_dataclass(o):
        return dataclasses.asdict(o)
    raise TypeError(repr(o))


def load_state(path, cfg=None, **engine_kw):
    """Resume a run from :func:`save_state`: a new Engine (``engine_kw`` as for initialize) holding the
    snapshot's population at its generation.  ``cfg`` defaults to the snapshot's configuration."""
    import json
    with np.load(path) as z:
        meta = json.loads(bytes(z["meta"]).decode())
        snap = {"format": meta["format"], "generation": meta["generation"], "config": meta["config"],
                "X": z["X"], "F": z["F"], "ideal": z["ideal"]}
    if cfg is None:
        c = dict(meta["config"])
        c["variation"] = VariationConfig(**c["variation"])
        if c.get("reference_points") is not None:
            c["reference_points"] = tuple(c["reference_points"])
        cfg = RunConfig(**c)
    eng = Engine(cfg, **engine_kw)
    eng.restore(snap)
    return _state(eng, {})


__all__ = ["RunConfig", "RunState", "Engine", "LocalShards", "initialize", "step", "run", "validate",
           "build_reference_set", "run_collective", "save_state", "load_state"]
