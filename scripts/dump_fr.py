"""Save the merged objectives (and the running ideal) of a late generation for host-side analysis
(dominance structure, sub-tile box classification, lattice-association certificate rates).
Usage: dump_fr.py [gens] [problem n m d] [sort]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 30
problem, n, m, d = (sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 \
    else ("DTLZ2", 10000, 5, 14)
sort = sys.argv[6] if len(sys.argv) > 6 else "auto"
cfg = engine.RunConfig(problem=problem, n=n, m=m, d=d, generations=gens, seed=0)
e = engine.Engine(cfg, sort=sort)
for _ in range(gens):
    e.step()
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
tag = f"{problem.lower()}_n{n}_m{m}_g{gens}"
np.save(f"gpurun_out/fr_{tag}.npy", e.FR[e.cur ^ 1].cpu().numpy())
np.save(f"gpurun_out/ideal_{tag}.npy", e.ideal.cpu().numpy())
print(e.info_dict())
