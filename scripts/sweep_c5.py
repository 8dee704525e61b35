"""C5: DTLZ1-7 x m x N sweep -- generations/s and IGD (population size vs quality).

BASELINE.json configs[4] / SURVEY.md 8(d) C5 (the paper's large-population
experiment).  For every (problem, m, n): G generations on
one GPU (bit-matrix sort where it fits, streamed sort beyond), device-timed
per generation after 3 warm-up generations, then IGD of the final
population against 10^4 points of the true front (metrics.igd on the GPU).

  python scripts/sweep_c5.py --problems DTLZ2,DTLZ7 --m 3,5,8,10 --n 1000,16000,256000 --gens 20
Prints one JSON line per configuration.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine, metrics  # noqa: E402


def d_for(problem, m):
    k = {"DTLZ1": 5, "DTLZ7": 20}.get(problem, 10)      # the suite's customary k = d - m + 1
    return m + k - 1


def run_one(problem, m, n, gens, seed=0, ref_points=10_000):
    cfg = engine.RunConfig(problem=problem, n=n, m=m, d=d_for(problem, m), generations=gens, seed=seed)
    t0 = time.time()
    eng = engine.Engine(cfg)
    torch.cuda.synchronize()
    setup = time.time() - t0
    for _ in range(3):
        eng.step()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(gens):
        eng.step()
    ev[1].record()
    ev[1].synchronize()
    ms = ev[0].elapsed_time(ev[1]) / gens
    pf = metrics.dtlz_pf_sample(problem, m, ref_points).astype("float32")
    q = metrics.igd(eng.F, pf)
    info = eng.info_dict()
    return {"problem": problem, "m": m, "n": n, "d": cfg.d, "w": eng.w,
            "sort": "bits" if eng.sort_mode == 0 else "stream", "generations": gens + 3,
            "ms_per_generation": round(ms, 4), "generations_per_s": round(1e3 / ms, 3), "igd": q,
            "setup_s": round(setup, 2), "last": {k: info[k] for k in ("l", "k", "nfronts", "survivors")}}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--problems", default="DTLZ1,DTLZ2,DTLZ3,DTLZ4,DTLZ5,DTLZ6,DTLZ7")
    p.add_argument("--m", default="3,5,8,10")
    p.add_argument("--n", default="1000,4000,16000,64000")
    p.add_argument("--gens", type=int, default=20)
    a = p.parse_args()
    for prob in a.problems.split(","):
        for m in map(int, a.m.split(",")):
            for n in map(int, a.n.split(",")):
                n += n % 2
                try:
                    print(json.dumps(run_one(prob, m, n, a.gens)), flush=True)
                except Exception as e:  # record and continue the sweep
                    print(json.dumps({"problem": prob, "m": m, "n": n, "error": repr(e)}), flush=True)
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
