"""C4 generation timeline: per-generation wall / device time and GPU busy fraction from the torch
profiler's CUPTI kernel records (no nsys in the image).  Usage: python scripts/c4_timeline.py [host|device] [n]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2504_06067_b200 import engine  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "host"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
poll = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = engine.RunConfig(problem="DTLZ7", n=n, m=3, d=22, generations=20, seed=0)
eng = engine.Engine(cfg, sort="stream", host_fronts=(mode == "host"), poll=poll)
eng._auto_fronts = False
for _ in range(3):
    eng.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(5):
    eng.step()
e1.record()
e1.synchronize()
wall = (time.perf_counter() - t0) / 5
dev = e0.elapsed_time(e1) / 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        eng.step()
    torch.cuda.synchronize()
import ctypes  # noqa: E402
from paper_2504_06067_b200 import _lib  # noqa: E402
off = ctypes.c_int64(0)
_lib.check(_lib.lib().mo_stream_stats_offset(n, 3, eng.w, eng.sort_mode, eng.shard_count, ctypes.byref(off)), "stats")
st = eng.ws[off.value: off.value + 32].view(torch.int64).cpu().tolist()
print(json.dumps({"count_pairs_le": st[0], "count_pairs_full": st[1], "dec_pairs_le": st[2], "dec_pairs_full": st[3]}))
ks = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = {}
for e in ks:
    a = agg.setdefault(e.name, [0, 0.0])
    a[0] += 1
    a[1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
tot = sum(v[1] for v in agg.values())
print(json.dumps({"mode": mode, "n": n, "poll": poll, "wall_ms": wall * 1e3, "device_ms": dev,
                  "kernel_ms_per_gen": tot / 2, "nfronts": eng.info_dict()["nfronts"]}))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {v[1]/2:9.3f} ms  {v[0]/2:6.1f}x  {k[:90]}")
