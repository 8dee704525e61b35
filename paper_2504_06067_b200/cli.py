"""Command line (the reference's ``manyobj`` script):

  python -m paper_2504_06067_b200.cli run --config plan.yaml --out results.csv [--seeds 0,1,2]
  python -m paper_2504_06067_b200.cli summarize results.csv
  python -m paper_2504_06067_b200.cli compare --problem DTLZ2 --m 3 --d 12 --sizes 800,3200 [--reps 3]

``run`` reads an ExperimentPlan from a YAML key-value file (fields of bench.ExperimentPlan).  Exit
code 0 on success; 2 for a bad configuration / input (ConfigError), 3 for any other failure.
``compare`` prints one JSON row per population size: the GPU batched engine's mean
per-generation time against the scalar Alg. 1 back-end (or ``--against batched-cpu``) and the ratio.
The CPU back-ends are timed only; see bench.compare_backends.
"""
import argparse
import json
import sys

from .errors import ConfigError


def _load_plan(path, out, seeds):
    import yaml

    from .bench import ExperimentPlan
    with open(path) as f:
        d = yaml.safe_load(f) or {}
    if not isinstance(d, dict):
        raise ConfigError("config", "expected a key-value mapping")
    fields = ExperimentPlan.__dataclass_fields__
    unknown = set(d) - set(fields)
    if unknown:
        raise ConfigError("config", f"unknown keys {sorted(unknown)}")
    for k in ("problems", "sizes", "generations", "seeds", "hv_ref"):
        if k in d and d[k] is not None and not isinstance(d[k], (list, tuple)):
            d[k] = [d[k]]
        if k in d and d[k] is not None:
            d[k] = tuple(d[k])
    if out:
        d["out"] = out
    if seeds:
        d["seeds"] = tuple(int(s) for s in seeds.split(","))
    return ExperimentPlan(**d)


def main(argv=None):
    p = argparse.ArgumentParser(prog="manyobj")
    sub = p.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--out")
    r.add_argument("--seeds")
    r.add_argument("--backend", default="batched")
    r.add_argument("--time-limit", type=float)
    s = sub.add_parser("summarize")
    s.add_argument("csv")
    c = sub.add_parser("compare")
    c.add_argument("--problem", default="DTLZ2")
    c.add_argument("--m", type=int, default=3)
    c.add_argument("--d", type=int, default=12)
    c.add_argument("--sizes", default="92")
    c.add_argument("--reps", type=int, default=1)
    c.add_argument("--generations", type=int, default=5)
    c.add_argument("--against", default="oracle")
    c.add_argument("--seed", type=int, default=0)
    a = p.parse_args(argv)
    try:
        if a.cmd == "run":
            if a.backend != "batched":
                raise ConfigError("backend", "only the batched GPU back-end is available")
            plan = _load_plan(a.config, a.out, a.seeds)
            if a.time_limit:
                import dataclasses
                plan = dataclasses.replace(plan, time_limit_s=a.time_limit)
            from .bench import run_plan
            print(run_plan(plan))
        elif a.cmd == "compare":
            from .bench import compare_backends
            try:
                sizes = tuple(int(x) for x in a.sizes.split(","))
            except ValueError:
                raise ConfigError("sizes", f"comma-separated integers expected, got {a.sizes!r}") from None
            for row in compare_backends(a.problem, a.m, a.d, sizes, a.reps, a.generations,
                                        ("batched", a.against), a.seed):
                print(json.dumps(row))
        else:
            from .bench import summarize
            print(json.dumps(summarize(a.csv), indent=1))
        return 0
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 -- CLI boundary: report the category, nonzero exit
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
