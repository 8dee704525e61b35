"""Eager vs graph timing of one C3 generation and of the niche phase, per association mode."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import _lib, engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
cfg = engine.RunConfig(problem="DTLZ3", n=n, m=10, d=19, generations=30, seed=0)
e = engine.Engine(cfg, sort="bits")
for _ in range(6):
    e.step()
torch.cuda.synchronize()
for rep in range(3):
    prof = {}
    e.step(profile=prof)
    torch.cuda.synchronize()
    print("profile", {k: round(v * 1e3, 3) for k, v in prof.items()}, flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    e.step()
    torch.cuda.synchronize()
    print("eager step ms", round((time.perf_counter() - t0) * 1e3, 3), flush=True)
