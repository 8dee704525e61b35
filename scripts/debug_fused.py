import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_06067_b200 as M
from paper_2504_06067_b200 import _lib
from oracle.manyobj_ref import dominance as Odom
rs = np.random.default_rng(0)
for m, R in [(5, 600), (5, 2000), (3, 600), (3, 2000), (6, 3000)]:
    F = rs.random((R, m)).astype(np.float32)
    cfg = M.engine.RunConfig(problem="DTLZ2", n=R // 2, m=m, d=m + 9, generations=1, seed=0)
    eng = M.engine.Engine(cfg, sort="stream")
    eng.FR[eng.cur].copy_(torch.from_numpy(F))
    _lib.check(_lib.lib().mo_step_phases(eng._args[eng.cur], _lib.PHASE_SORT, _lib.stream_ptr()), "sort")
    torch.cuda.synchronize()
    r = eng.ranks.cpu().numpy()
    want = Odom.non_dominated_sort(F, stop_at=R // 2)
    bad = np.nonzero(r != want)[0]
    print(m, R, "mismatch", len(bad), eng.info_dict(), "want l", Odom.split_fronts(want, R // 2).l, bad[:5], r[bad[:5]], want[bad[:5]], flush=True)
