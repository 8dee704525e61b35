"""Time a few generations of a large workload with the streamed sort (per-phase)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_06067_b200 import engine

wl = dict(c4=("DTLZ7", 3, 22, 1_000_000), c3=("DTLZ3", 10, 19, 100_000), c2=("DTLZ2", 5, 14, 10_000),
          m3_100k=("DTLZ7", 3, 22, 100_000), m3_300k=("DTLZ7", 3, 22, 300_000))
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sort = sys.argv[3] if len(sys.argv) > 3 else "stream"
poll = int(sys.argv[4]) if len(sys.argv) > 4 else 4
kind, m, d, n = wl[name]
cfg = engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=0)
t0 = time.time()
eng = engine.Engine(cfg, sort=sort, poll=poll)
torch.cuda.synchronize()
print(f"init {time.time() - t0:.2f}s w={eng.w}", flush=True)
for g in range(gens):
    prof = {}
    t0 = time.time()
    eng.step(profile=prof)
    torch.cuda.synchronize()
    dt = time.time() - t0
    extra = {}
    if eng.sort_mode == 1:
        import ctypes
        from paper_2504_06067_b200 import _lib
        off = ctypes.c_int64(0)
        _lib.lib().mo_stream_stats_offset(n, m, eng.w, eng.sort_mode, eng.shard_count, ctypes.byref(off))
        st = eng.ws[off.value: off.value + 32].view(torch.int64).cpu().tolist()
        extra = {"pairs_count_le": st[0], "pairs_count_full": st[1], "pairs_dec_le": st[2], "pairs_dec_full": st[3]}
    print(json.dumps({"gen": g, "wall_s": round(dt, 4), **{k: round(v, 5) for k, v in prof.items()},
                      **eng.info_dict(), **extra}), flush=True)
