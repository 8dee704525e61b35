"""Phase trace of the persistent kernels for an arbitrary config: trace_cfg.py PROBLEM m d n gens"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import _lib, engine  # noqa: E402

prob, m, d, n, gens = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
cfg = engine.RunConfig(problem=prob, n=n, m=m, d=d, generations=gens, seed=0)
eng = engine.Engine(cfg)
off = int(_lib.lib().mo_trace_offset(cfg.n, cfg.m, eng.w))
for g in range(gens):
    eng.ws[off: off + 512].zero_()
    prof = {}
    eng.step(profile=prof)
    torch.cuda.synchronize()
    if g >= gens - 2:
        print(f"gen {g}: " + " ".join(f"{k}={v * 1e3:.3f}" for k, v in prof.items()))
        print("   " + " ".join(f"{k}={v:.1f}" for k, v in eng.trace().items()))
        print("   ", eng.info_dict())
