"""Phase trace (globaltimer marks of the persistent kernels) of one graph-replayed generation after a warm
run: trace_graph.py [workload] [warm]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_06067_b200 import _lib, engine  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 500
cfg = engine.RunConfig(problem=wl["problem"], n=wl["n"], m=wl["m"], d=wl["d"], generations=warm + 10, seed=0)
eng = engine.Engine(cfg, graph=True)
eng.replay(warm)
off = int(_lib.lib().mo_trace_offset(cfg.n, cfg.m, eng.w))
for _ in range(3):
    eng.ws[off: off + 512].zero_()
    eng.replay(1)
    torch.cuda.synchronize()
    print(" ".join(f"{k}={v:.1f}" for k, v in eng.trace().items()))
