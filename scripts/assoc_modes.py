"""Graph-replay generations/s of a config with the lattice association (prune=True) vs the tensor-core
filtered full scan (prune=False); checks the runs stay bit-identical.  assoc_modes.py [PROBLEM m d n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

prob, m, d, n = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else \
    ("DTLZ2", 5, 14, 10000)
ref = None
for prune in (True, False):
    cfg = engine.RunConfig(problem=prob, n=n, m=m, d=d, generations=700, seed=0)
    eng = engine.Engine(cfg, graph=True, prune=prune)
    eng.replay(300)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.replay(300)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 300
    X = eng.X.clone()
    same = None if ref is None else bool(torch.equal(ref, X))
    ref = X if ref is None else ref
    print(f"prune={prune} lattice={eng.lattice is not None} hmma={eng.zfrag is not None}: {ms * 1e3:.1f} us/gen "
          f"= {1e3 / ms:.0f} gen/s; identical: {same}")
