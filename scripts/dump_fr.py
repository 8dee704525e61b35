"""Save the merged objectives (and the running ideal) of a late C2 generation for host-side analysis
(sub-tile box classification, lattice-association certificate rates).  Usage: dump_fr.py [gens]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = engine.RunConfig(problem="DTLZ2", n=10000, m=5, d=14, generations=gens, seed=0)
e = engine.Engine(cfg)
for _ in range(gens):
    e.step()
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/fr_c2_g{gens}.npy", e.FR[e.cur ^ 1].cpu().numpy())
np.save(f"gpurun_out/ideal_c2_g{gens}.npy", e.ideal.cpu().numpy())
print(e.info_dict())
