"""Generation time along a long run (CUDA-graph replays, windows of 20 generations): does the
per-generation cost drift as the population converges?  Usage: python scripts/long_run.py c3 300"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

SHAPES = {"c1": ("DTLZ1", 92, 3, 7), "c2": ("DTLZ2", 10000, 5, 14), "c3": ("DTLZ3", 100000, 10, 19)}
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 300
p, n, m, d = SHAPES[name]
eng = engine.Engine(engine.RunConfig(problem=p, n=n, m=m, d=d, generations=G, seed=0), graph=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = []
for g0 in range(0, G, 20):
    torch.cuda.synchronize()
    e0.record()
    eng.replay(20)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    info = eng.info_dict()
    out.append({"gens": [g0, g0 + 20], "ms_per_gen": round(ms, 4), "l": info["l"], "level": info["level"],
                "nfronts": info["nfronts"], "error": info["error"]})
    print(json.dumps(out[-1]), flush=True)
