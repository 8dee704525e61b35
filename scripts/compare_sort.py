"""Bits vs streamed sort: device ms per generation for (problem, m, n) configurations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

cases = [c.split(":") for c in sys.argv[1].split(",")]   # e.g. DTLZ7:3:64000,DTLZ4:3:128000
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for prob, m, n in cases:
    m, n = int(m), int(n)
    out = {"problem": prob, "m": m, "n": n}
    for sort in ("bits", "stream", "stream_dev"):
        cfg = engine.RunConfig(problem=prob, n=n, m=m, d=m + (19 if prob == "DTLZ7" else 9), generations=gens, seed=0)
        if sort == "bits" and 2 * n > 300_000:
            continue
        eng = engine.Engine(cfg, sort=sort.replace("_dev", ""), host_fronts=(sort == "stream"))
        for _ in range(3):
            eng.step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(gens):
            eng.step()
        e1.record()
        e1.synchronize()
        out[sort + "_ms"] = round(e0.elapsed_time(e1) / gens, 3)
        out[sort + "_fronts"] = eng.info_dict()["nfronts"]
        del eng
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
