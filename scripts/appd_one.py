"""One Appendix D configuration (DTLZ3, N=800, d=1000, m from argv), eager generations: for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
eng = engine.Engine(engine.RunConfig(problem="DTLZ3", n=800, m=m, d=1000, generations=8, seed=0))
for _ in range(8):
    eng.step()
torch.cuda.synchronize()
print(eng.info_dict())
