"""Wide objective counts (16 < m <= 512, Appendix D: DTLZ3 m = 4 ... 512, N = 800, d = 1000):
the runtime-m kernels (k_dom_rank_wide, k_prep's runtime-m extremes + block-parallel FP64 solve with the
system in global memory for m > 64, k_assoc_wide, k_assoc_final_rt) against the oracle, op by op and
generation by generation (state injection)."""
import numpy as np
import pytest

from oracle.manyobj_ref import dominance as Odom
from oracle.manyobj_ref import engine as Oeng
from oracle.manyobj_ref import niche as Oniche
from oracle.manyobj_ref import problems as Oprob
from oracle.manyobj_ref import refpoints as Oref
from oracle.manyobj_ref import rng as Orng
from oracle.manyobj_ref import variation as Ovar

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2504_06067_b200 as pkg
    from paper_2504_06067_b200 import _lib
    _lib.lib()
    return pkg


def np_(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("R,m,kind", [(700, 17, "rand"), (1300, 24, "ties"), (600, 64, "rand"),
                                      (520, 200, "ties"), (300, 512, "rand"), (1600, 40, "dtlz")])
def test_ranked_bits_wide(M, R, m, kind):
    """k_dom_rank_wide (objective chunks of 8) == the dominance matrix, every word below wend, hasdom."""
    rs = np.random.default_rng(R + m)
    if kind == "rand":
        F = rs.random((R, m))
    elif kind == "ties":
        F = rs.integers(0, 2, size=(R, m)).astype(np.float64)
        F[: R // 4] = F[R // 4: R // 2]                      # duplicates
    else:
        X = rs.random((R, m + 9)).astype(np.float32)
        F = Oprob.dtlz_eval(Oprob.ContinuousProblem("DTLZ2", m, m + 9), X)
    F = F.astype(np.float32)
    ps = M.dominance.presort(F)
    perm = np_(ps["perm"])
    we = np_(ps["wend"])
    bits, hasdom = M.dominance.dominance_bits_sorted(ps, poison=True, method="ranked")
    D = Odom.dominance_matrix(F[perm])
    dense = np_(M.dominance.unpack_bits(bits, R))
    for j in range(R):
        lim = min(R, we[j] * 32)
        assert np.array_equal(dense[:lim, j], D[:lim, j]), (m, j)
        assert not D[lim:, j].any()
    assert np.array_equal(np_(hasdom).astype(bool), D.any(axis=0))


def _front_instance(seed, R, m, kind="DTLZ3"):
    rs = np.random.default_rng(seed)
    d = m + 9
    X = rs.random((R, d)).astype(np.float32)
    F = Oprob.dtlz_eval(Oprob.ContinuousProblem(kind, m, d), X).astype(np.float32)
    n = R // 2
    ranks = Odom.non_dominated_sort(F, stop_at=n)
    return F, ranks, Odom.split_fronts(ranks, n), n


@pytest.mark.parametrize("seed,R,m", [(0, 400, 17), (1, 600, 33), (2, 300, 64), (3, 500, 65), (4, 1200, 100),
                                      (5, 1000, 512)])
def test_normalize_wide(M, seed, R, m):
    """Runtime-m extreme points (top-2 ASF), the block-parallel FP64 solve (global system for m > 64)."""
    F, ranks, sp, n = _front_instance(seed, R, m)
    cand = (ranks <= sp.l) & (ranks != Odom.DROPPED)
    ideal0 = np.full(m, np.inf, np.float32)
    gen = 3
    pos_pop = Orng.positions(R, seed, gen, Orng.STREAM_POP_SHUFFLE)
    Fn, ideal, a, ext, singular = Oniche.normalize_objectives(F, ideal0, cand, pos_pop)
    gFn, gideal, gicpt = M.niche.normalize_objectives(F, ideal0, ranks.astype(np.int32), sp.l, seed, gen)
    assert np.array_equal(np_(gideal), ideal)
    assert np.array_equal(np_(gicpt), a), (singular, np_(gicpt)[:4], a[:4])
    assert np.array_equal(np_(gFn)[cand], Fn[cand])


@pytest.mark.parametrize("seed,R,m,w_target", [(0, 400, 17, 200), (1, 1600, 40, 800), (2, 800, 128, 300),
                                               (3, 1600, 512, 800)])
def test_associate_wide(M, seed, R, m, w_target):
    F, ranks, sp, n = _front_instance(seed, R, m)
    cand = (ranks <= sp.l) & (ranks != Odom.DROPPED)
    Z = Oref.reference_points(m, w_target)
    zh = Oref.unit_directions(Z)
    gen = 4
    pos_pop = Orng.positions(R, seed, gen, Orng.STREAM_POP_SHUFFLE)
    pos_ref = Orng.positions(len(Z), seed, gen, Orng.STREAM_REF_SHUFFLE)
    Fn, *_ = Oniche.normalize_objectives(F, np.full(m, np.inf, np.float32), cand, pos_pop)
    pi, d = Oniche.associate_canonical(Fn, zh, pos_ref, np.flatnonzero(cand))
    Fn_in = np.where(cand[:, None], Fn, 0).astype(np.float32)
    gpi, gd = M.niche.associate_canonical(Fn_in, zh, ranks.astype(np.int32), sp.l, seed, gen)
    assert np.array_equal(np_(gpi)[cand], pi[cand])
    assert np.array_equal(np_(gd)[cand], d[cand])


@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ3", 200, 17, 30, 4), ("DTLZ2", 300, 32, 50, 4),
                                             ("DTLZ3", 800, 64, 1000, 3), ("DTLZ1", 160, 65, 80, 3),
                                             ("DTLZ3", 800, 128, 1000, 2), ("DTLZ3", 800, 512, 1000, 2)])
def test_engine_wide_state_injection(M, kind, n, m, d, gens):
    """Appendix D shapes: every generation the oracle's selection on the GPU's merged objectives picks
    exactly the GPU's survivors (X, F, ideal bit-equal; l and k equal)."""
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=5)
    ocfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=5)
    eng = M.engine.Engine(cfg)
    assert eng.sort_mode == M._lib.SORT_BITS
    for g in range(gens):
        st = Oeng.RunState(eng.generation, np_(eng.X).copy(), np_(eng.F).copy(), np_(eng.ideal).copy(),
                           Oref.unit_directions(eng.Z), eng.Z)
        cur = eng.cur
        eng.step()
        O = np_(eng.XR[cur][n:]).copy()
        FO = np_(eng.FR[cur][n:]).copy()
        assert np.allclose(O, Ovar.vary(st.X, ocfg.variation, 5, g), rtol=1e-6, atol=1e-7)
        nxt = Oeng.step(st, ocfg, offspring=(O, FO))
        info = eng.info_dict()
        assert info["survivors"] == n and info["error"] == 0
        assert info["l"] == nxt.info["l"] and info["k"] == nxt.info["k"]
        assert np.array_equal(np_(eng.X), nxt.X), f"generation {g}"
        assert np.array_equal(np_(eng.F), nxt.F)
        assert np.array_equal(np_(eng.ideal), nxt.ideal)


def test_engine_wide_graph_equals_eager(M):
    cfg = M.engine.RunConfig(problem="DTLZ3", n=800, m=100, d=1000, generations=4, seed=2)
    a = M.engine.Engine(cfg)
    for _ in range(4):
        a.step()
    b = M.engine.Engine(cfg, graph=True)
    b.replay(4)
    import torch
    torch.cuda.synchronize()
    assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F) and torch.equal(a.ideal, b.ideal)
