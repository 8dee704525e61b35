"""C2 niche-phase time with the full-scan association vs the lattice at several radii."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_06067_b200 import engine
wl = dict(c2=("DTLZ2", 5, 14, 10000), m5_100k=("DTLZ2", 5, 14, 100000), m4_10k=("DTLZ2", 4, 13, 10000))
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kind, m, d, n = wl[name]
cfg = engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=20, seed=0)
for prune, r in [(False, 0), (True, 2), (True, 3), (True, 4)]:
    eng = engine.Engine(cfg, prune=prune, prune_r=r)
    for _ in range(10):
        eng.step()
    prof = {}
    for _ in range(10):
        eng.step(profile=prof)
    print(json.dumps({"wl": name, "prune": prune, "r": r, "t_niche_ms": round(prof["t_niche"] / 10 * 1e3, 4),
                      "fallback": eng.info_dict()["assoc_fallback"], "survivors": eng.info_dict()["survivors"]}))
