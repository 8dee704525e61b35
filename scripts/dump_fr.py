"""Save the merged objectives of a late C2 generation (analysis of sub-tile box classification)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_06067_b200 import engine
cfg = engine.RunConfig(problem="DTLZ2", n=10000, m=5, d=14, generations=30, seed=0)
e = engine.Engine(cfg)
for _ in range(30):
    e.step()
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/fr_c2.npy", e.FR[e.cur ^ 1].cpu().numpy())
