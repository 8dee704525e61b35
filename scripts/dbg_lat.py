import sys, time
sys.path.insert(0, '.')
import torch
import paper_2504_06067_b200 as M
for (kind, m, d, n) in [("DTLZ5", 2, 11, 1000), ("DTLZ7", 3, 22, 3000), ("DTLZ2", 4, 13, 4000), ("DTLZ2", 5, 14, 10000)]:
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=2, seed=6)
    e = M.engine.Engine(cfg, prune=True)
    t = time.time()
    e.step(); torch.cuda.synchronize()
    print(kind, m, "ok", round(time.time() - t, 3), e.info_dict()["assoc_fallback"], flush=True)
