"""Per-phase globaltimer trace of the persistent kernels (engine.trace()) at C1 / C2 / C3 shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

SHAPES = {"c1": ("DTLZ1", 92, 3, 7), "c2": ("DTLZ2", 10000, 5, 14), "c3": ("DTLZ3", 100000, 10, 19)}
for name in sys.argv[1:] or ["c1", "c2"]:
    p, n, m, d = SHAPES[name]
    eng = engine.Engine(engine.RunConfig(problem=p, n=n, m=m, d=d, generations=100, seed=0))
    for _ in range(30):
        eng.step()
    acc = {}
    for _ in range(20):
        eng.step()
        torch.cuda.synchronize()
        for k, v in eng.trace().items():
            acc.setdefault(k, []).append(v)
    print(json.dumps({"shape": name, **{k: round(sorted(v)[len(v) // 2], 2) for k, v in acc.items()}}))
