"""The paper's Appendix D objective scan on the B200 engine: DTLZ3, N = 800, d = 1000, m = 4 ... 512
(PAPER.md:395-420), per-generation runtime.  Device-timed CUDA-graph replays (100 generations after 3
warm-up ones, as the paper's 100-generation runs); m > 16 runs the runtime-m kernels.  With --cpu, the
CPU restatement of the reference (oracle/manyobj_ref numpy + oracle/c quadratic stages, all host cores)
is timed on 2 generations per m beside it (the reference arm; bench harness use only)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

PAPER_TENSOR_S = {4: 4.334e-3, 8: 4.624e-3, 16: 5.083e-3, 32: 6.514e-3, 64: 8.103e-3, 128: 1.016e-2,
                  256: 2.348e-2, 512: 3.199e-2}
PAPER_CPU_S = {4: 9.219e-1, 8: 1.061, 16: 4.722e-1, 32: 8.684e-1, 64: 4.784e-1, 128: 9.282e-1, 256: 2.012,
               512: 3.918}
cpu = "--cpu" in sys.argv
for m, paper_s in PAPER_TENSOR_S.items():
    n, d = 800, 1000
    cfg = engine.RunConfig(problem="DTLZ3", n=n, m=m, d=d, generations=103, seed=0)
    eng = engine.Engine(cfg, graph=True)
    eng.replay(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    eng.replay(100)
    e1.record()
    e1.synchronize()
    s = e0.elapsed_time(e1) / 100 / 1e3
    info = eng.info_dict()
    rec = {"problem": "DTLZ3", "m": m, "d": d, "n": n, "w": eng.w, "s_per_generation": s,
           "generations_per_s": 1 / s, "last_l": info["l"], "error": info["error"],
           "paper_tensornsga3_s": paper_s, "ratio_vs_paper_tensornsga3": paper_s / s,
           "paper_nsga3_cpu_s": PAPER_CPU_S[m]}
    if cpu:
        from oracle import c as oc
        from oracle.manyobj_ref import engine as Oeng
        from oracle.manyobj_ref import refpoints as Oref
        ocfg = Oeng.RunConfig(problem="DTLZ3", n=n, m=m, d=d, generations=2, seed=0)
        st = Oeng.RunState(eng.generation, eng.X.cpu().numpy().copy(), eng.F.cpu().numpy().copy(),
                           eng.ideal.cpu().numpy().copy(), Oref.unit_directions(eng.Z), eng.Z)
        # oracle/c restates the quadratic stages for m <= 16; beyond, the numpy restatement alone
        acc = oc.accel(threads=len(os.sched_getaffinity(0))) if m <= 16 else {}
        per = []
        for _ in range(2):
            t0 = time.perf_counter()
            st = Oeng.step(st, ocfg, **acc)
            per.append(time.perf_counter() - t0)
        rec["cpu_reference_s_per_generation"] = min(per)
        rec["gpu_vs_cpu_reference"] = min(per) / s
    print(json.dumps(rec), flush=True)
