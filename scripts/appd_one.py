"""One Appendix D configuration (DTLZ3, N=800, d=1000, m from argv) for launch lists: 3 eager warm-up
generations, then argv[2] generations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = engine.Engine(engine.RunConfig(problem="DTLZ3", n=800, m=m, d=1000, generations=g + 3, seed=0))
for _ in range(3 + g):
    eng.step()
torch.cuda.synchronize()
print(eng.info_dict(), eng.trace())
