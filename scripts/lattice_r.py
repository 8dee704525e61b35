"""Graph-replay generations/s of C2 for several lattice radii (prune_r) and a check that the runs stay
bit-identical (the certified association is exact for every radius).  Usage: lattice_r.py [r ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

radii = [int(x) for x in sys.argv[1:]] or [0, 1]
ref = None
for r in radii:
    cfg = engine.RunConfig(problem="DTLZ2", n=10000, m=5, d=14, generations=800, seed=0)
    eng = engine.Engine(cfg, graph=True, prune_r=r)
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
    print(f"prune_r={r}: {ms * 1e3:.1f} us/gen = {1e3 / ms:.0f} gen/s; identical to first: {same}; "
          f"info {eng.info_dict()}")
