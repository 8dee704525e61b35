"""Per-phase globaltimer trace of the persistent kernels over a few generations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_06067_b200 import engine  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
cfg = engine.RunConfig(problem=wl["problem"], n=wl["n"], m=wl["m"], d=wl["d"], generations=100, seed=0)
eng = engine.Engine(cfg)
for g in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    eng.ws[int(__import__("paper_2504_06067_b200._lib", fromlist=["x"]).lib().mo_trace_offset(cfg.n, cfg.m, eng.w)):].__getitem__(slice(0, 512)).zero_()
    prof = {}
    eng.step(profile=prof)
    torch.cuda.synchronize()
    tr = eng.trace()
    print(f"gen {g}: phases(ms) " + " ".join(f"{k}={v*1e3:.3f}" for k, v in prof.items()))
    print("   " + " ".join(f"{k}={v:.1f}" for k, v in tr.items()))
    print("   ", eng.info_dict())
