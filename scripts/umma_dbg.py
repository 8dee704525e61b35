"""Timing experiment for k_assoc_umma's pipeline (MO_UMMA_DEBUG): the C3 association kernel time with
the epilogue's candidate work off (1), the MMAs off (2), both (3).  Results invalid under the flags."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import _lib, engine  # noqa: E402

cfg = engine.RunConfig(problem="DTLZ3", n=100000, m=10, d=19, generations=30, seed=0)
e = engine.Engine(cfg, sort="bits")
for _ in range(8):
    e.step()
torch.cuda.synchronize()
L = _lib.lib()
a = e._args[e.cur]
# time the NICHE_ASSOC phase alone on the current merged buffer (after PREP of the same state)
_lib.check(L.mo_step_phases(a, _lib.PHASE_VARY | _lib.PHASE_SORT, _lib.stream_ptr()), "vs")
_lib.check(L.mo_niche_phases(a, _lib.NICHE_PREP, _lib.stream_ptr()), "prep")
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(L.mo_niche_phases(a, _lib.NICHE_ASSOC, _lib.stream_ptr()), "assoc")
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("MO_UMMA_DEBUG", "0"), sorted(ts))
