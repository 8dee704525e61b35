"""Experiment harness (the reference's ``bench`` module).

* :class:`ExperimentPlan` -- a grid of RunConfigs (problems x sizes x generations x seeds),
  repetitions, a per-cell time limit and an output path.
* :func:`run_plan` -- runs every cell on the GPU engine and writes one CSV row per generation with
  the SPEC schema (fingerprint, seed, generation, igd, hv_raw, hv_normalized, t_variation, t_sort,
  t_niche, t_eval, timed_out).  IGD (GPU, FP64) against 10^4 front points; HV on the GPU: exact for
  m <= 3, Monte-Carlo (``hv_samples``, fixed seed) for m > 3; hv_normalized = hv_raw / HV_max with
  HV_max = prod(ref - 0.9 f^min) over the true-front sample (Appendix E Eqs. 3-5).  The CSV is
  written atomically (temp file + rename).
* :func:`summarize` -- per fingerprint: mean, standard deviation and 95 % t-interval of the final IGD /
  HV and of the per-generation runtime (generation 1 excluded: one-time setup).
* :func:`compare_backends` -- SPEC.md:686-694 (Table I's analogue): per population size, the mean
  per-generation time of two back-ends on identical seeds and their ratio.  "batched" is this package's
  GPU engine; the scalar Alg. 1 back-end ("oracle") is the CPU restatement under ``oracle/`` -- test
  infrastructure that the product path never calls -- and is only *timed* here, loaded lazily by
  module name (``MANYOBJ_ORACLE``, default ``oracle.manyobj_ref.engine``) when a comparison names it.
"""
import csv
import dataclasses
import hashlib
import json
import math
import os
import tempfile
import time
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

COLUMNS = ("fingerprint", "seed", "generation", "igd", "hv_raw", "hv_normalized", "t_variation", "t_sort",
           "t_niche", "t_eval", "timed_out")


@dataclass(frozen=True)
class ExperimentPlan:
    """SPEC.md:658-661."""
    problems: tuple = ("DTLZ2",)
    m: int = 3
    d: int = 12
    sizes: tuple = (92,)
    generations: tuple = (100,)
    seeds: tuple = (0,)
    repetitions: int = 1
    time_limit_s: float = 600.0
    out: str = "results.csv"
    ref_points: int = 10_000
    hv_ref: tuple = None            # reference point for HV (default 1.1 x the front's nadir sample)
    hv_samples: int = 100_000

    def cells(self):
        for p in self.problems:
            for n in self.sizes:
                for g in self.generations:
                    yield p, n, g

    def validate(self):
        if self.repetitions < 1:
            raise ConfigError("repetitions", "must be >= 1")
        if not (self.problems and self.sizes and self.generations and self.seeds):
            raise ConfigError("plan", "the grid has no cell")


def fingerprint(cfg):
    """Stable hash of a RunConfig's fields (seed excluded: it is its own column)."""
    d = dataclasses.asdict(cfg)
    d.pop("seed", None)
    return hashlib.sha1(json.dumps(d, sort_keys=True, default=str).encode()).hexdigest()[:12]


def _metrics(F, ref, hv_ref, hv_ideal, hv_samples, seed):
    from . import metrics
    q = metrics.igd(F, ref)
    hv = metrics.hv(F, hv_ref, samples=hv_samples, seed=seed)
    vol = float(np.prod(np.asarray(hv_ref) - hv_ideal))
    return q, hv, hv / vol if vol > 0 else 0.0


def run_plan(plan, progress=None):
    """Run every (cell, seed, repetition); write the CSV atomically; return the output path."""
    import torch

    from . import engine, metrics
    plan.validate()
    rows = []
    for prob, n, gens in plan.cells():
        pf = metrics.dtlz_pf_sample(prob, plan.m, plan.ref_points).astype(np.float32)
        hv_ref = tuple(plan.hv_ref) if plan.hv_ref else tuple(1.1 * pf.max(axis=0))
        hv_ideal = 0.9 * pf.astype(np.float64).min(axis=0)
        for seed in plan.seeds:
            for _ in range(plan.repetitions):
                cfg = engine.RunConfig(problem=prob, n=n, m=plan.m, d=plan.d, generations=gens, seed=seed)
                fp = fingerprint(cfg)
                state = engine.initialize(cfg)
                t0 = time.time()
                for g in range(1, gens + 1):
                    state = engine.step(state, cfg, profile=True)
                    prof = state.timings
                    timed_out = (time.time() - t0) > plan.time_limit_s
                    q, hv, hvn = _metrics(state.F, pf, hv_ref, hv_ideal, plan.hv_samples, seed)
                    rows.append({"fingerprint": fp, "seed": seed, "generation": g, "igd": q, "hv_raw": hv,
                                 "hv_normalized": hvn,
                                 **{k: prof.get(k, 0.0) for k in ("t_variation", "t_sort", "t_niche", "t_eval")},
                                 "timed_out": int(timed_out)})
                    state = dataclasses.replace(state, timings={})
                    if timed_out:
                        break
                torch.cuda.synchronize()
                if progress:
                    progress(prob, n, gens, seed)
    return write_rows(rows, plan.out)


def write_rows(rows, path):
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, suffix=".tmp")
    try:
        with os.fdopen(fd, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=COLUMNS)
            w.writeheader()
            for r in rows:
                w.writerow({k: r[k] for k in COLUMNS})
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return path


def _tci(x):
    """mean, sample std, 95 % t-interval half width."""
    from scipy import stats
    x = np.asarray(x, np.float64)
    mean = float(x.mean())
    if x.size < 2:
        return mean, 0.0, 0.0
    sd = float(x.std(ddof=1))
    return mean, sd, float(stats.t.ppf(0.975, x.size - 1) * sd / math.sqrt(x.size))


def read_rows(path):
    rows = []
    with open(path, newline="") as f:
        r = csv.DictReader(f)
        if tuple(r.fieldnames or ()) != COLUMNS:
            raise ConfigError("csv", f"unexpected header {r.fieldnames}")
        for lineno, row in enumerate(r, start=2):
            try:
                rows.append({"fingerprint": row["fingerprint"], "seed": int(row["seed"]),
                             "generation": int(row["generation"]),
                             **{k: float(row[k]) for k in COLUMNS[3:10]}, "timed_out": int(row["timed_out"])})
            except (TypeError, ValueError) as e:
                raise ConfigError("csv", f"line {lineno}: {e}") from None
    return rows


def summarize(path):
    """per fingerprint, statistics over seeds of the final IGD / HV and of the
    per-generation runtime (generation 1 excluded)."""
    rows = read_rows(path)
    out = {}
    by = {}
    for r in rows:
        by.setdefault(r["fingerprint"], []).append(r)
    for fp, rs in by.items():
        final = {}
        times = []
        for r in rs:
            key = r["seed"]
            if key not in final or r["generation"] > final[key]["generation"]:
                final[key] = r
            if r["generation"] > 1:
                times.append(r["t_variation"] + r["t_sort"] + r["t_niche"] + r["t_eval"])
        fin = list(final.values())
        out[fp] = {"runs": len(fin),
                   "igd": _tci([r["igd"] for r in fin]),
                   "hv_normalized": _tci([r["hv_normalized"] for r in fin]),
                   "s_per_generation": _tci(times) if times else (float("nan"), 0.0, 0.0)}
    return out


# ------------------------------------------------------------------ compare_backends

def _gpu_backend(cfg, generations):
    """Per-generation seconds of the GPU engine (generation 1 excluded: one-time setup)."""
    import torch

    from . import engine
    state = engine.initialize(cfg)
    per = []
    for _ in range(generations):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        state = engine.step(state)
        state.engine.check_errors(block=True)
        per.append(time.perf_counter() - t0)
    return per


def _cpu_backend(niching):
    def run(cfg, generations):
        import importlib
        O = importlib.import_module(os.environ.get("MANYOBJ_ORACLE", "oracle.manyobj_ref.engine"))
        ocfg = O.RunConfig(problem=cfg.problem, n=cfg.n, m=cfg.m, d=cfg.d, generations=generations,
                           seed=cfg.seed, backend=niching)
        st = O.initialize(ocfg)
        per = []
        for _ in range(generations):
            t0 = time.perf_counter()
            st = O.step(st, ocfg)
            per.append(time.perf_counter() - t0)
        return per
    return run


BACKENDS = {"batched": _gpu_backend,
            # the CPU restatements (timing only): Alg. 1 scalar niching, and the batched CPU loop
            "oracle": _cpu_backend("oracle"),
            "batched-cpu": _cpu_backend("batched")}


def compare_backends(problem="DTLZ2", m=3, d=12, sizes=(92,), reps=1, generations=5,
                     backends=("batched", "oracle"), seed=0):
    """for each population size, the mean per-generation time (generation 1 excluded)
    of ``backends[0]`` and ``backends[1]`` over ``reps`` identical-seed runs (seeds seed..seed+reps-1),
    and the ratio t(backends[1]) / t(backends[0]) (the speed-up of the first over the second).
    Returns one row per size."""
    from . import engine
    if reps < 1 or generations < 2:
        raise ConfigError("reps", "reps >= 1 and generations >= 2 (generation 1 is excluded)")
    if len(backends) != 2 or any(b not in BACKENDS for b in backends):
        raise ConfigError("backend", f"two of {sorted(BACKENDS)}")
    if not sizes:
        raise ConfigError("sizes", "at least one population size")
    rows = []
    for n in sizes:
        times = {}
        for b in backends:
            per = []
            for r in range(reps):
                cfg = engine.RunConfig(problem=problem, n=int(n), m=m, d=d, generations=generations,
                                       seed=seed + r)
                engine.validate(cfg)
                per.extend(BACKENDS[b](cfg, generations)[1:])
            times[b] = _tci(per)
        t0, t1 = times[backends[0]][0], times[backends[1]][0]
        rows.append({"problem": problem, "m": m, "d": d, "n": int(n), "reps": reps,
                     "generations": generations,
                     f"s_per_gen_{backends[0]}": t0, f"ci95_{backends[0]}": times[backends[0]][2],
                     f"s_per_gen_{backends[1]}": t1, f"ci95_{backends[1]}": times[backends[1]][2],
                     "ratio": t1 / t0 if t0 > 0 else float("inf")})
    return rows


__all__ = ["ExperimentPlan", "COLUMNS", "fingerprint", "run_plan", "write_rows", "read_rows", "summarize",
           "compare_backends", "BACKENDS"]
