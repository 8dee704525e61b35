"""The paper's Table I configuration on the B200 engine: DTLZ3, m=6, d=500, per-generation runtime vs n
(BASELINE.md).  Device-timed CUDA-graph replays, 100 generations after 3 warm-up ones
(the paper: 100 generations, 31 repetitions, mean per-generation time)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

PAPER_TENSOR_S = {50: 1.120e-3, 100: 1.135e-3, 200: 1.121e-3, 400: 1.243e-3, 800: 1.493e-3, 1600: 2.063e-3,
                  3200: 4.886e-3, 6400: 1.575e-2, 12800: 5.966e-2}
for n, paper_s in PAPER_TENSOR_S.items():
    cfg = engine.RunConfig(problem="DTLZ3", n=n, m=6, d=500, generations=103, seed=0)
    eng = engine.Engine(cfg, graph=True)
    eng.replay(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    eng.replay(100)
    e1.record()
    e1.synchronize()
    s = e0.elapsed_time(e1) / 100 / 1e3
    print(json.dumps({"problem": "DTLZ3", "m": 6, "d": 500, "n": n, "w": eng.w, "s_per_generation": s,
                      "generations_per_s": 1 / s, "paper_tensornsga3_v100_s": paper_s,
                      "ratio_vs_paper_v100": paper_s / s}), flush=True)
