import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2504_06067_b200 as M
ref = M.metrics.dtlz_pf_sample("DTLZ2", 3, 10_000).astype(np.float32)
for gens in (200, 400):
    vals = []
    for s in range(10):
        cfg = M.engine.RunConfig(problem="DTLZ2", n=92, m=3, d=12, generations=gens, seed=s)
        _, st = M.engine.run(cfg, record=False, graph=True)
        vals.append(M.metrics.igd(st.F, ref))
    print(gens, np.round(vals, 4), np.median(vals))
# floor: the reference directions themselves (on the sphere)
Z = M.refpoints.reference_points(3, 92); zh = Z / np.linalg.norm(Z, axis=1, keepdims=True)
print("floor (ideal 91-point set):", M.metrics.igd(zh.astype(np.float32), ref))
