"""Debug: DTLZ7 n=600 state-injection mismatch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2504_06067_b200 as M
from oracle.manyobj_ref import dominance as Odom, engine as Oeng, refpoints as Oref

kind, n, m, d, gens = "DTLZ7", 600, 3, 22, 6
for trial in range(3):
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=17)
    ocfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=17)
    eng = M.engine.Engine(cfg)
    for g in range(gens):
        st = Oeng.RunState(g, eng.X.cpu().numpy().copy(), eng.F.cpu().numpy().copy(), eng.ideal.cpu().numpy().copy(),
                           Oref.unit_directions(eng.Z), eng.Z)
        cur = eng.cur
        eng.step()
        O = eng.XR[cur][n:].cpu().numpy().copy()
        FO = eng.FR[cur][n:].cpu().numpy().copy()
        FR = eng.FR[cur].cpu().numpy().copy()
        nxt = Oeng.step(st, ocfg, offspring=(O, FO))
        info = eng.info_dict()
        ranks_o = Odom.non_dominated_sort(FR, stop_at=n)
        g_r = eng.ranks.cpu().numpy()
        ok = info["l"] == nxt.info["l"] and info["k"] == nxt.info["k"]
        print(trial, g, info, nxt.info, "ok" if ok else "MISMATCH")
        if not ok:
            l = info["l"]
            print(" oracle front sizes", np.bincount(ranks_o[ranks_o != Odom.DROPPED]))
            sel = (g_r < l) & (g_r >= 0)
            print(" gpu <l count", sel.sum(), "oracle <l", (ranks_o < l).sum())
            diff = np.nonzero((ranks_o < l) != ((g_r < l)))[0]
            print(" diff rows", diff[:10], ranks_o[diff[:10]], g_r[diff[:10]])
            # rerun the sort alone on FR
            r2, i2 = M.dominance.non_dominated_sort(FR, stop_at=n, return_info=True)
            print(" op-level bits sort equal oracle:", np.array_equal(r2.cpu().numpy(), ranks_o))
            ps = M.dominance.presort(FR)
            bits, hasdom = M.dominance.dominance_bits_sorted(ps)
            perm = ps["perm"].cpu().numpy()
            D = Odom.dominance_matrix(FR[perm])
            dense = M.dominance.unpack_bits(bits, 2 * n).cpu().numpy()
            we = ps["wend"].cpu().numpy()
            bad = 0
            for j in range(2 * n):
                lim = min(2 * n, we[j] * 32)
                if not np.array_equal(dense[:lim, j], D[:lim, j]) or D[lim:, j].any():
                    bad += 1
            print(" sorted bits bad rows:", bad)
            break
