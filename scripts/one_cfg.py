"""Run one configuration eagerly for ncu launch lists: one_cfg.py PROBLEM m n d gens"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

prob, m, n, d, gens = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
eng = engine.Engine(engine.RunConfig(problem=prob, n=n, m=m, d=d, generations=gens, seed=0))
for _ in range(gens):
    eng.step()
torch.cuda.synchronize()
print(eng.info_dict())
