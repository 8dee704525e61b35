"""Run a few eager C2 generations (for ncu). Usage: python scripts/profile_step.py [workload] [gens] [warm]
(warm: that many earlier generations run first, e.g. to profile the steady state; skip them in ncu with
--launch-skip warm*kernels_per_generation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_06067_b200 import engine  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 4
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = engine.RunConfig(problem=wl["problem"], n=wl["n"], m=wl["m"], d=wl["d"], generations=gens + warm, seed=0)
eng = engine.Engine(cfg)
for _ in range(warm):
    eng.step()
torch.cuda.synchronize()
for _ in range(gens):
    eng.step()
torch.cuda.synchronize()
print(eng.info_dict())
