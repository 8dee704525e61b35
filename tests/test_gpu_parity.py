"""GPU (sm_100a) parity against the CPU oracle, through the C-ABI library.

Bit-exact: permutations, initial population, dominance bits, ranks, split,
ideal, intercepts, Fn, pi, d, survivor sets.  Tolerance (north star: 1e-5
relative in FP32): offspring and objectives, which the GPU computes in FP64
and rounds once (so they agree to ~1 ulp in practice; tested at rtol 1e-6).
"""
import numpy as np
import pytest
import torch

from conftest import examples
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
    _lib.lib()  # fails loudly without the library / device
    return pkg


def np_(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ L1 / RNG

@pytest.mark.parametrize("n", [1, 2, 3, 17, 184, 1000, 20000])
def test_permutation_bit_exact(M, n):
    for seed, gen, stream in [(0, 0, 5), (123456789012, 7, 6), (5, 99, 2)]:
        perm = M.variation.permutation(n, seed, gen, stream)
        assert np.array_equal(np_(perm), Orng.permutation(n, seed, gen, stream))


def test_init_population_bit_exact(M):
    X = M.variation.init_population(92, 7, 11)
    assert np.array_equal(np_(X), Oeng.initial_population(92, 7, 11))


@pytest.mark.parametrize("kind", Oprob.KINDS)
def test_dtlz_eval_matches_oracle(M, kind):
    rs = np.random.default_rng(1)
    for m, d in [(3, 7), (5, 14), (10, 19), (3, 22)]:
        X = rs.random((257, d)).astype(np.float32)
        X[:5] = np.round(X[:5])                   # exact 0/1 corners
        P = M.problems.ContinuousProblem(kind, m, d)
        got = np_(M.problems.dtlz_eval(P, X))
        want = Oprob.dtlz_eval(Oprob.ContinuousProblem(kind, m, d), X.astype(np.float64)).astype(np.float32)
        assert np.allclose(got, want, rtol=1e-6, atol=1e-7), (kind, m, d)


def test_dtlz_golden(M):
    from paper_2504_06067_b200 import errors
    for ex in examples({"dtlz_point", "dtlz_domain"}):
        P = M.problems.ContinuousProblem(ex["kind"], ex["m"], ex["d"])
        if "error" in ex:
            with pytest.raises(errors.DomainError):
                M.problems.dtlz_eval(P, np.array([ex["x"]], np.float32))
        else:
            assert np.allclose(np_(M.problems.dtlz_eval(P, np.array([ex["x"]], np.float32)))[0], ex["out"],
                               atol=1e-6)


@pytest.mark.parametrize("kind,m,d", [("DTLZ1", 3, 7), ("DTLZ2", 5, 14), ("DTLZ3", 10, 19), ("DTLZ7", 3, 22),
                                      ("DTLZ4", 4, 9), ("DTLZ5", 4, 9), ("DTLZ6", 4, 9)])
def test_vary_eval_matches_oracle(M, kind, m, d):
    rs = np.random.default_rng(3)
    n = 256
    X = rs.random((n, d)).astype(np.float32)
    X[:4, :2] = 0.0
    X[4:8, :2] = 1.0
    cfg = M.variation.VariationConfig()
    P = M.problems.ContinuousProblem(kind, m, d)
    Xo, Fo = M.variation.vary_eval(P, X, cfg, seed=77, generation=5)
    want_X = Ovar.vary(X, Ovar.VariationConfig(), 77, 5)
    assert np.allclose(np_(Xo), want_X, rtol=1e-6, atol=1e-7)
    want_F = Oprob.dtlz_eval(Oprob.ContinuousProblem(kind, m, d), np_(Xo).astype(np.float64)).astype(np.float32)
    assert np.allclose(np_(Fo), want_F, rtol=1e-6, atol=1e-7)
    # bit-exact fraction: FP64 internals round to the same FP32 almost always
    assert (np_(Xo) == want_X).mean() > 0.999


# ----------------------------------------------------------------- dominance

def _instances():
    rs = np.random.default_rng(21)
    for R, m in [(1, 2), (2, 2), (31, 3), (32, 3), (255, 2), (256, 5), (257, 3), (700, 4), (1100, 10),
                 (600, 1)]:
        yield rs.random((R, m)).astype(np.float32)
        yield rs.integers(0, 3, size=(R, m)).astype(np.float32)       # ties + duplicates


def test_dominance_matrix_bit_exact(M):
    for F in _instances():
        got = np_(M.dominance.dominance_matrix(F))
        assert np.array_equal(got, Odom.dominance_matrix(F)), F.shape


def test_dominance_with_valid_mask(M):
    rs = np.random.default_rng(5)
    F = rs.integers(0, 4, size=(300, 3)).astype(np.float32)
    valid = rs.random(300) < 0.7
    got = np_(M.dominance.dominance_matrix(F, valid))
    D = Odom.dominance_matrix(F)
    D &= valid[:, None] & valid[None, :]
    assert np.array_equal(got, D)
    r = np_(M.dominance.non_dominated_sort(F, valid))
    assert np.array_equal(r, Odom.non_dominated_sort(F, valid))


@pytest.mark.parametrize("method", ["ranked", "pairwise"])
def test_sorted_path_bits(M, method):
    """Engine sort path: S-ordered buckets, bits of every row up to wend, hasdom flags."""
    rs = np.random.default_rng(12)
    signed0 = rs.integers(-1, 2, size=(520, 3)).astype(np.float32)
    signed0[rs.random((520, 3)) < 0.5] *= -0.0                         # -0 == +0 ties
    cases = [rs.random((700, 3)), rs.integers(0, 3, size=(600, 4)), rs.random((1300, 5)),
             np.repeat(rs.random((300, 2)), 3, axis=0), rs.random((257, 10)), signed0,
             rs.integers(0, 2, size=(900, 16)), np.round(rs.random((1100, 12)) * 3) / 3,
             np.full((300, 6), 0.5)]
    for F in cases:
        F = F.astype(np.float32)
        R, m = F.shape
        ps = M.dominance.presort(F)
        perm = np_(ps["perm"])
        assert sorted(perm.tolist()) == list(range(R))
        S = F[:, 0].copy()
        for k in range(1, m):
            S = (S + F[:, k]).astype(np.float32)
        SS = np_(ps["SS"])
        assert np.array_equal(SS, S[perm]) and np.array_equal(np_(ps["FS"]), F[perm])
        # order inside a bucket is free ...
        we = np_(ps["wend"])
        # ... but no later position outside p's bucket may have S <= S[p]
        for p in range(R):
            later = np.arange((we[p]) * 32, R)
            # (an S = -0 bucket precedes the S = +0 one: FP-equal sums, no dominance either way)
            eq = SS[later] == SS[p]
            assert (SS[later] >= SS[p]).all() and not (eq & (np.signbit(SS[later]) == np.signbit(SS[p]))).any()
        bmin, bmax = np_(ps["blkmin"]), np_(ps["blkmax"])
        for b in range(len(bmin)):
            blk = SS[b * 256:(b + 1) * 256]
            assert bmin[b] == blk.min() and bmax[b] == blk.max()
        bits, hasdom = M.dominance.dominance_bits_sorted(ps, poison=True, method=method)
        D = Odom.dominance_matrix(F[perm])                      # D[i][j]: i dominates j (position space)
        dense = np_(M.dominance.unpack_bits(bits, R))
        for j in range(R):
            lim = min(R, we[j] * 32)
            assert np.array_equal(dense[:lim, j], D[:lim, j]), (F.shape, j)
            assert not D[lim:, j].any()
        assert np.array_equal(np_(hasdom).astype(bool), D.any(axis=0))


@pytest.mark.parametrize("method", ["ranked", "pairwise"])
def test_sorted_bits_bucket_straddling_fast_tile(M, method):
    """A S-bucket straddling a block boundary whose tile is fast: the i rows' words of the later block
    lie below wend and must be written (zeros), not left stale (regression: stale bits from the previous
    generation made the peel see phantom dominators)."""
    rs = np.random.default_rng(44)
    hit = 0
    for trial in range(40):
        low = rs.random((255, 3)).astype(np.float32) * 3.0               # S < 9
        high = 11.0 + rs.random((255, 3)).astype(np.float32) * 1000.0    # S > 33
        pair = np.array([[10.2, 0.0, 0.0], [0.0, 10.2 + 1e-5 * (1 + trial % 5), 0.0]], np.float32)
        ext = np.array([[0.0, 0.0, 0.0]], np.float32)
        F = np.concatenate([low[:254], ext, pair, high, [[65536.0, 0.0, 0.0]]]).astype(np.float32)
        F = F[rs.permutation(len(F))]
        R = F.shape[0]
        ps = M.dominance.presort(F)
        perm = np_(ps["perm"])
        we = np_(ps["wend"])
        bmin, bmax = np_(ps["blkmin"]), np_(ps["blkmax"])
        hit += int(we[255] > 8 and bmax[0] < bmin[1])
        bits, hasdom = M.dominance.dominance_bits_sorted(ps, poison=True, method=method)
        D = Odom.dominance_matrix(F[perm])
        dense = np_(M.dominance.unpack_bits(bits, R))
        for j in range(R):
            lim = min(R, we[j] * 32)
            assert np.array_equal(dense[:lim, j], D[:lim, j]), (trial, j)
        r = np_(M.dominance.non_dominated_sort(F, stop_at=R // 2))
        assert np.array_equal(r, Odom.non_dominated_sort(F, stop_at=R // 2))
    assert hit > 0, "construction never produced a straddling fast tile"


def test_ranked_bits_nan_rows(M):
    """A row with a NaN objective dominates nothing and is dominated by nothing (the oracle's
    (A <= B).all() & (A < B).any() with IEEE compares); the rank-mask kernel keeps that."""
    rs = np.random.default_rng(9)
    F = rs.integers(0, 3, size=(700, 4)).astype(np.float32)
    F[rs.random((700, 4)) < 0.02] = np.nan
    ps = M.dominance.presort(F)
    perm = np_(ps["perm"])
    we = np_(ps["wend"])
    bits, hasdom = M.dominance.dominance_bits_sorted(ps, poison=True, method="ranked")
    D = Odom.dominance_matrix(F[perm])
    dense = np_(M.dominance.unpack_bits(bits, 700))
    for j in range(700):
        lim = min(700, we[j] * 32)
        assert np.array_equal(dense[:lim, j], D[:lim, j]), j


def test_ranked_bits_large_many_blocks(M):
    """Multi-block sweep (items spanning several J blocks), C3-like m = 10 and a tie-heavy m = 5."""
    rs = np.random.default_rng(21)
    for F in (rs.random((9000, 10)).astype(np.float32),
              (np.round(rs.random((7000, 5)) * 6) / 6).astype(np.float32)):
        R = F.shape[0]
        ps = M.dominance.presort(F)
        a, ha = M.dominance.dominance_bits_sorted(ps, method="ranked")
        b, hb = M.dominance.dominance_bits_sorted(ps, method="pairwise")
        we = torch.as_tensor(np_(ps["wend"])).cuda().long()
        cols = torch.arange(a.shape[1], device="cuda")[None, :]
        live = cols < we[:, None]
        assert torch.equal(a[live], b[live]) and torch.equal(ha, hb)


def test_nds_bit_exact(M):
    for F in _instances():
        assert np.array_equal(np_(M.dominance.non_dominated_sort(F)), Odom.non_dominated_sort(F)), F.shape


def test_nds_stop_at(M):
    rs = np.random.default_rng(8)
    for R, m in [(184, 3), (2000, 3), (4000, 5)]:
        F = rs.random((R, m)).astype(np.float32)
        n = R // 2
        ranks, info = M.dominance.non_dominated_sort(F, stop_at=n, return_info=True)
        want = Odom.non_dominated_sort(F, stop_at=n)
        assert np.array_equal(np_(ranks), want)
        sp = M.dominance.split_from_info(info)
        wsp = Odom.split_fronts(want, n)
        assert (sp.l, sp.selected_count, sp.k) == (wsp.l, wsp.selected_count, wsp.k)


def test_dominance_golden(M):
    from paper_2504_06067_b200 import errors
    for ex in examples({"dominates", "dominance_matrix", "non_dominated_sort", "split_fronts"}):
        op = ex["op"]
        if op == "dominates":
            if "error" in ex:
                with pytest.raises(errors.ShapeError):
                    M.dominance.dominates(ex["a"], ex["b"])
            else:
                assert M.dominance.dominates(ex["a"], ex["b"]) == ex["out"]
        elif op == "dominance_matrix":
            assert np_(M.dominance.dominance_matrix(np.array(ex["F"], np.float32))).tolist() == ex["out"]
        elif op == "non_dominated_sort":
            assert np_(M.dominance.non_dominated_sort(np.array(ex["F"], np.float32))).tolist() == ex["out"]
        else:
            ranks = np.concatenate([np.full(s, i) for i, s in enumerate(ex["sizes"])]).astype(np.int32)
            if "error" in ex:
                with pytest.raises(errors.InfeasibleSplitError):
                    M.dominance.split_fronts(ranks, ex["n"])
            else:
                sp = M.dominance.split_fronts(ranks, ex["n"])
                assert [sp.l, sp.selected_count, sp.k] == ex["out"]


def test_nds_infeasible(M):
    from paper_2504_06067_b200 import errors
    F = np.random.default_rng(0).random((10, 3)).astype(np.float32)
    valid = np.zeros(10, bool)
    valid[:3] = True
    _, info = M.dominance.non_dominated_sort(F, valid, stop_at=5, return_info=True)
    with pytest.raises(errors.InfeasibleSplitError):
        M.dominance.split_from_info(info)


# -------------------------------------------------------------------- niche

def _front_instance(seed, R, m, kind="DTLZ2"):
    rs = np.random.default_rng(seed)
    X = rs.random((R, m + 4)).astype(np.float32)
    F = Oprob.dtlz_eval(Oprob.ContinuousProblem(kind, m, m + 4), X).astype(np.float32)
    n = R // 2
    ranks = Odom.non_dominated_sort(F, stop_at=n)
    sp = Odom.split_fronts(ranks, n)
    return F, ranks, sp, n


@pytest.mark.parametrize("seed,R,m", [(0, 184, 3), (1, 2000, 5), (2, 4000, 3), (3, 3000, 10), (4, 1000, 8)])
def test_normalize_bit_exact(M, seed, R, m):
    F, ranks, sp, n = _front_instance(seed, R, m)
    cand = (ranks <= sp.l) & (ranks != Odom.DROPPED)
    ideal0 = np.full(m, np.inf, np.float32)
    gen = 3
    pos_pop = Orng.positions(R, seed, gen, Orng.STREAM_POP_SHUFFLE)
    Fn, ideal, a, ext, singular = Oniche.normalize_objectives(F, ideal0, cand, pos_pop)
    gFn, gideal, gicpt = M.niche.normalize_objectives(F, ideal0, ranks.astype(np.int32), sp.l, seed, gen)
    assert np.array_equal(np_(gideal), ideal)
    assert np.array_equal(np_(gicpt), a)
    assert np.array_equal(np_(gFn)[cand], Fn[cand])


def test_normalize_golden(M):
    for ex in examples({"normalize"}):
        F = np.array(ex["F"], np.float32)
        ideal = None if ex["ideal"] is None else np.array(ex["ideal"], np.float32)
        Fn, idl, a = M.niche.normalize_objectives(F, ideal)
        assert np.allclose(np_(Fn), ex["out"], atol=1e-6)
        if "intercepts" in ex:
            assert np.allclose(np_(a), ex["intercepts"])


@pytest.mark.parametrize("seed,R,m,w_target", [(0, 184, 3, 91), (1, 2000, 5, 1000), (2, 5000, 3, 2500),
                                              (3, 3000, 10, 1500), (4, 1024, 2, 512)])
def test_associate_bit_exact(M, seed, R, m, w_target):
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
    assert (np_(gpi)[~cand] == -1).all()


@pytest.mark.parametrize("seed,R,m,w_target", [(0, 184, 3, 91), (1, 2000, 5, 1000), (2, 6000, 3, 3000),
                                              (5, 2000, 3, 40), (6, 1500, 8, 700)])
def test_niche_select_bit_exact(M, seed, R, m, w_target):
    F, ranks, sp, n = _front_instance(seed, R, m)
    Z = Oref.reference_points(m, w_target)
    zh = Oref.unit_directions(Z)
    gen = 2
    sel, info = Oniche.select(F, ranks, sp, np.full(m, np.inf, np.float32), zh, seed, gen)
    if info["skipped"]:
        pytest.skip("instance needed no niching")
    gsel, granks, ginfo = M.niche.niche_select(info["pi"].astype(np.int32), info["d"], ranks.astype(np.int32),
                                               sp, n, len(Z), seed, gen)
    assert np.array_equal(np_(gsel), sel)
    assert int(np_(gsel).sum()) == n
    assert ginfo["NEAREST"] == len(info["nearest"])


@pytest.mark.parametrize("seed,R,w,f0,f1,n", [(0, 40000, 8, 0, 30000, 20000), (1, 40000, 16, 5000, 30000, 20000),
                                               (2, 12000, 3, 3000, 6000, 6000), (3, 200000, 40, 20000, 150000, 100000)])
def test_niche_select_crowded_levels(M, seed, R, w, f0, f1, n):
    """Crowded niches (thousands of members per reference point, as DTLZ3 m=10 late in a run): the water
    level lies beyond k_select's 1024-bin histogram window (grid-cooperative 32-ary level search) and the
    partially taken buckets hold thousands of candidates (radix top-t select)."""
    rs = np.random.default_rng(seed)
    ranks = np.full(R, 2, np.int32)
    ranks[:f0] = 0
    ranks[f0:f0 + f1] = 1 if f0 else 0
    rs.shuffle(ranks)
    sp = Odom.split_fronts(ranks, n)
    assert not sp.infeasible if hasattr(sp, "infeasible") else True
    p = 1.0 / np.arange(1, w + 1)
    pi = rs.choice(w, size=R, p=p / p.sum()).astype(np.int32)
    d = rs.random(R).astype(np.float32)
    cand = ranks <= sp.l
    pi[~cand] = -1
    d[~cand] = 0
    F = rs.random((R, 3)).astype(np.float32)
    zh = np.ones((w, 3), np.float32) / np.sqrt(3)
    gen = 7
    sel, info = Oniche.select(F, ranks, sp, np.full(3, np.inf, np.float32), zh, seed, gen,
                              associate_fn=lambda Fn, z, pos_ref, rows: (pi, d))
    assert not info["skipped"]
    gsel, granks, ginfo = M.niche.niche_select(pi, d, ranks, sp, n, w, seed, gen)
    assert ginfo["LEVEL"] >= 1024, ginfo            # the instance exercises the search beyond the window
    assert np.array_equal(np_(gsel), sel)
    assert int(np_(gsel).sum()) == n
    assert ginfo["NEAREST"] == len(info["nearest"])


# ------------------------------------------------------------------- engine

def _gpu_state_to_oracle(eng):
    return Oeng.RunState(eng.generation, np_(eng.X).copy(), np_(eng.F).copy(), np_(eng.ideal).copy(),
                         Oref.unit_directions(eng.Z), eng.Z)


@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ1", 92, 3, 7, 30), ("DTLZ2", 1000, 5, 14, 6),
                                             ("DTLZ3", 400, 10, 19, 4), ("DTLZ7", 600, 3, 22, 6),
                                             ("DTLZ4", 200, 4, 13, 6), ("DTLZ5", 200, 4, 13, 6),
                                             ("DTLZ6", 200, 3, 12, 6)])
def test_engine_step_state_injection(M, kind, n, m, d, gens):
    """Every generation: the oracle's selection on the GPU's merged objectives picks the GPU's survivors."""
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=17)
    ocfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=17)
    eng = M.engine.Engine(cfg)
    X0 = Oeng.initial_population(n, d, 17)
    assert np.array_equal(np_(eng.X), X0)
    skipped = niched = 0
    for g in range(gens):
        st = _gpu_state_to_oracle(eng)
        cur = eng.cur
        eng.step()
        # offspring the GPU produced (rows n..2n of the merged buffer it just consumed)
        O = np_(eng.XR[cur][n:]).copy()
        FO = np_(eng.FR[cur][n:]).copy()
        want_O = Ovar.vary(st.X, ocfg.variation, 17, g)
        assert np.allclose(O, want_O, rtol=1e-6, atol=1e-7)
        nxt = Oeng.step(st, ocfg, offspring=(O, FO))
        info = eng.info_dict()
        assert info["survivors"] == n
        assert info["l"] == nxt.info["l"] and info["k"] == nxt.info["k"]
        assert np.array_equal(np_(eng.X), nxt.X), f"generation {g}"
        assert np.array_equal(np_(eng.F), nxt.F)
        assert np.array_equal(np_(eng.ideal), nxt.ideal)
        skipped += info["skipped"]
        niched += 1 - info["skipped"]
    assert niched > 0


def test_engine_graph_equals_eager(M):
    cfg = M.engine.RunConfig(problem="DTLZ2", n=500, m=5, d=14, generations=8, seed=4)
    a = M.engine.Engine(cfg)
    for _ in range(8):
        a.step()
    b = M.engine.Engine(cfg, graph=True)
    b.replay(8)
    torch.cuda.synchronize()
    assert a.generation == b.generation == 8
    assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F) and torch.equal(a.ideal, b.ideal)


def test_engine_determinism(M):
    cfg = M.engine.RunConfig(problem="DTLZ1", n=92, m=3, d=7, generations=20, seed=9)
    h1, s1 = M.engine.run(cfg)
    h2, s2 = M.engine.run(cfg)
    assert h1 == h2 and torch.equal(s1.X, s2.X)


def test_engine_c2_full_size_properties(M):
    """C2 (DTLZ2 m=5 d=14 n=10k): size-independent invariants of one generation at full size."""
    cfg = M.engine.RunConfig(problem="DTLZ2", n=10000, m=5, d=14, generations=3, seed=0)
    eng = M.engine.Engine(cfg)
    for _ in range(3):
        eng.step()
        info = eng.info_dict()
        assert info["survivors"] == 10000 and info["error"] == 0
    F = eng.F
    assert torch.isfinite(F).all() and (eng.X >= 0).all() and (eng.X <= 1).all()
    # ranks of the last step against the oracle NDS of the same merged objectives
    FR = np_(eng.FR[eng.cur ^ 1]).copy()
    ranks = Odom.non_dominated_sort(FR, stop_at=10000)
    l = Odom.split_fronts(ranks, 10000).l
    g = np_(eng.ranks)
    assert info["l"] == l
    assert np.array_equal(g[ranks < l], ranks[ranks < l])
    assert np.isin(g[ranks == l], [l, l - 1]).all()
    assert (g[ranks == Odom.DROPPED] == Odom.DROPPED).all()


def test_engine_rejects_oracle_backend(M):
    from paper_2504_06067_b200 import errors
    with pytest.raises(errors.ConfigError) as ei:
        M.engine.initialize(M.engine.RunConfig(backend="oracle"))
    assert ei.value.field == "backend"


# ------------------------------------------------ broad state-injection sweep (all engine paths)

SWEEP = [(k, n, m, d, sort) for (k, n, m, d) in [("DTLZ2", 300, 2, 11), ("DTLZ1", 400, 3, 7), ("DTLZ7", 500, 4, 23),
                                                   ("DTLZ4", 300, 5, 14), ("DTLZ3", 300, 6, 15), ("DTLZ5", 200, 8, 17),
                                                   ("DTLZ6", 250, 10, 19), ("DTLZ2", 2000, 3, 12)]
         for sort in ("bits", "stream")]


@pytest.mark.parametrize("kind,n,m,d,sort", SWEEP)
def test_engine_sweep_state_injection(M, kind, n, m, d, sort):
    """m = 2 .. 10 (single- and two-layer reference sets, lattice pruning where it applies), both sort
    modes: every generation the oracle's selection on the GPU's merged objectives picks the GPU's
    survivors exactly."""
    gens = 3
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=23)
    ocfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=23)
    eng = M.engine.Engine(cfg, sort=sort, prune=True if m <= 5 and eng_prunable(m, n) else "auto")
    for g in range(gens):
        st = _gpu_state_to_oracle(eng)
        cur = eng.cur
        eng.step()
        O = np_(eng.XR[cur][n:]).copy()
        FO = np_(eng.FR[cur][n:]).copy()
        nxt = Oeng.step(st, ocfg, offspring=(O, FO))
        info = eng.info_dict()
        assert info["l"] == nxt.info["l"] and info["k"] == nxt.info["k"], (g, info)
        assert np.array_equal(np_(eng.X), nxt.X), f"generation {g}"
        assert np.array_equal(np_(eng.ideal), nxt.ideal)


def eng_prunable(m, n):
    from paper_2504_06067_b200 import refpoints
    return refpoints.choose_divisions(m, n)[1] == 0
