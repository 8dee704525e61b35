"""Structure of the C3 dominance bit-matrix at a late generation (design data for the peel / sweep):
dominators per row, nonzero 256-bit tiles per row, and -- for the rank-mask sweep -- how many objectives
a row j needs before the running AND over block I is empty (per-lane early exit).
Usage: bits_stats.py [gens] [problem n m d]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06067_b200 import _lib, engine  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 25
problem, n, m, d = (sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 \
    else ("DTLZ3", 100000, 10, 19)
cfg = engine.RunConfig(problem=problem, n=n, m=m, d=d, generations=gens, seed=0)
e = engine.Engine(cfg, sort="bits")
for _ in range(gens):
    e.step()
torch.cuda.synchronize()
R = 2 * n
W = int(_lib.lib().mo_bits_words_per_row(R))
nb = W // 8
bits = e.ws[: R * W * 4].view(torch.int32).view(R, W)          # layout: bits first (rows in presort order)
# the last step's presort permutation is not exported: the stats below are permutation-free per row
pc = torch.zeros(R, dtype=torch.int64, device="cuda")
nzt = torch.zeros(R, dtype=torch.int64, device="cuda")
for c0 in range(0, R, 4096):
    blk = bits[c0:c0 + 4096]
    x = blk.to(torch.int64) & 0xffffffff
    cnt = torch.zeros(blk.shape[0], W, dtype=torch.int64, device="cuda")
    for s in range(32):
        cnt += (x >> s) & 1
    pc[c0:c0 + 4096] = cnt.sum(1)
    nzt[c0:c0 + 4096] = (blk.view(-1, nb, 8) != 0).any(-1).sum(1)
q = torch.tensor([0.5, 0.9, 0.99, 1.0], device="cuda", dtype=torch.float64)
FR = e.FR[e.cur ^ 1]
out = {"R": R, "nb": nb, "info": e.info_dict(),
       "dominators_mean": pc.double().mean().item(), "dominators_q": torch.quantile(pc.double(), q).tolist(),
       "nonzero_tiles_mean": nzt.double().mean().item(), "nonzero_tiles_q": torch.quantile(nzt.double(), q).tolist(),
       "words_scanned_upper_bound_mean": W / 2}
# early exit: sample rows j; for each block I of 256 rows (in merged order, S-sorted below), the first
# objective count after which no i in I has a_i <= b_j in all objectives seen so far
F = FR.float()
S = F.sum(1)
order = torch.argsort(S)
FS = F[order]
g = torch.Generator(device="cuda").manual_seed(0)
js = torch.randint(0, R, (512,), device="cuda", generator=g)
need = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
for j in js.tolist():
    b = FS[j]
    le = (FS[:j] <= b)                       # rows before j in S order (the fast-tile side)
    if le.shape[0] == 0:
        continue
    acc = torch.cumprod(le.to(torch.int32), dim=1)          # prefix AND over objectives
    pad = (-le.shape[0]) % 256
    acc = torch.nn.functional.pad(acc, (0, 0, 0, pad)).view(-1, 256, m)
    alive = acc.any(1)                                      # (blocks, m): some i still <= after k+1 objs
    k_needed = alive.sum(1)                                  # objectives processed before it died (+1)
    k_needed = torch.clamp(k_needed + 1, max=m)
    need += torch.bincount(k_needed, minlength=m + 1)
out["objectives_needed_hist"] = need.tolist()
print(json.dumps(out))
