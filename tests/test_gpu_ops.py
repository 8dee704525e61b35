"""The op-level API on the GPU (k_ops.cu through the C-ABI): SPEC.md's worked examples
(tests/golden/spec_examples.json) and random instances against the oracle functions they restate
(oracle/manyobj_ref/batchcore.py, niche.py, variation.py) -- bit-exact for every index, count and
order; FP64 variation at 1e-12 (same operation order as the oracle, libdevice pow)."""
import numpy as np
import pytest
import torch

from conftest import examples
from oracle.manyobj_ref import batchcore as Ob
from oracle.manyobj_ref import dominance as Od
from oracle.manyobj_ref import niche as On
from oracle.manyobj_ref import rng as Orng
from oracle.manyobj_ref import variation as Ov

pytestmark = pytest.mark.gpu
INF = int(On.INF)


@pytest.fixture(scope="module")
def M():
    import paper_2504_06067_b200 as pkg
    from paper_2504_06067_b200 import _lib
    _lib.lib()
    return pkg


def np_(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ batchcore

@pytest.mark.parametrize("ex", examples({"step_mask"}), ids=lambda e: e["line"])
def test_step_mask_golden(M, ex):
    assert np_(M.batchcore.step_mask(ex["x"])).tolist() == ex["out"]


@pytest.mark.parametrize("ex", examples({"masked_argmin"}), ids=lambda e: e["line"])
def test_masked_argmin_golden(M, ex):
    from paper_2504_06067_b200 import errors
    if "error" in ex:
        with pytest.raises(getattr(errors, ex["error"])):
            M.batchcore.masked_argmin(ex["values"], ex["valid"])
    else:
        assert M.batchcore.masked_argmin(ex["values"], ex["valid"]) == ex["out"]


@pytest.mark.parametrize("ex", examples({"segment_count"}), ids=lambda e: e["line"])
def test_segment_count_golden(M, ex):
    assert np_(M.batchcore.segment_count(ex["labels"], ex["valid"], ex["segments"])).tolist() == ex["out"]


def test_batchcore_random_vs_oracle(M):
    from paper_2504_06067_b200 import errors
    rs = np.random.default_rng(0)
    for n in (1, 7, 1000, 300001):
        x = rs.integers(-3, 4, n).astype(np.float64)                  # many ties
        valid = rs.random(n) < 0.7
        valid[rs.integers(n)] = True
        assert np.array_equal(np_(M.batchcore.step_mask(x)), Ob.step_mask(x))
        assert M.batchcore.masked_argmin(x, valid) == Ob.masked_argmin(x, valid)
        assert M.batchcore.masked_argmin(x) == Ob.masked_argmin(x)
        lab = rs.integers(0, 50, n)
        assert np.array_equal(np_(M.batchcore.segment_count(lab, valid, 50)), Ob.segment_count(lab, valid, 50))
    with pytest.raises(errors.BoundsError):
        M.batchcore.segment_count([0, 5], None, 5)
    assert np_(M.batchcore.segment_count([0, 5], [1, 0], 5)).tolist() == [1, 0, 0, 0, 0]


# -------------------------------------------------------------------- niche

@pytest.mark.parametrize("ex", examples({"associate"}), ids=lambda e: e["line"])
def test_associate_golden(M, ex):
    pi, d = M.niche.associate(np.array(ex["D"], float), np.array(ex["valid"], bool))
    assert np_(pi).tolist() == ex["pi"]
    if "d" in ex:
        assert np.allclose(np_(d), ex["d"])


def test_associate_matrix_vs_oracle(M):
    rs = np.random.default_rng(1)
    D = rs.integers(0, 5, (513, 77)).astype(np.float64)
    valid = rs.random(513) < 0.8
    pi, d = M.niche.associate(D, valid)
    opi, od = On.associate(D, valid)
    assert np.array_equal(np_(pi), opi)
    assert np.array_equal(np.isnan(np_(d)), np.isnan(od)) and np.array_equal(np_(d)[valid], od[valid])


@pytest.mark.parametrize("ex", examples({"niche_counts"}), ids=lambda e: e["line"])
def test_niche_counts_golden(M, ex):
    rho, rho_p = M.niche.niche_counts(np.array(ex["pi"]), np.array(ex["ranks"]), ex["l"], ex["w"])
    want = [INF if v == "inf" else v for v in ex["rho"]]
    assert np_(rho).tolist() == want and np_(rho_p).tolist() == ex["rho_p"]


@pytest.mark.parametrize("ex", examples({"nearest"}), ids=lambda e: e["line"])
def test_nearest_golden(M, ex):
    pi, d, ranks = np.array(ex["pi"]), np.array(ex["d"], np.float32), np.array(ex["ranks"])
    rho, rho_p = M.niche.niche_counts(pi, ranks, ex["l"], ex["w"])
    pr, _, _ = M.niche.nearest_selection(pi, d, ranks, ex["l"], rho, rho_p, ex["k"], np.arange(len(pi)),
                                         np.arange(ex["w"]))
    assert sorted(np_(pr).tolist()) == ex["out"]


def test_build_cache_golden(M):
    ex = examples({"build_cache"})[0]
    pi, ranks = np.array(ex["pi"]), np.array(ex["ranks"])
    offs, cand = M.niche.build_cache(pi, ranks, ex["l"], ex["w"], np.arange(len(pi)), np.zeros(0, np.int64))
    offs, cand = np_(offs), np_(cand)
    j = ex["row"]
    assert cand[offs[j]:offs[j + 1]].tolist() == ex["out"]
    offs, cand = M.niche.build_cache(np.array([0, 0]), np.array([0, 0]), 0, 2, np.arange(2), np.zeros(0, np.int64))
    assert int(offs[2] - offs[1]) == 0                                 # no candidates -> empty row
    offs, cand = M.niche.build_cache(np.array([0, 0, 0]), np.zeros(3, int), 0, 1, np.arange(3), np.array([0]))
    assert np_(cand).tolist() == [1, 2]                                # nearest-taken candidate skipped


def test_batched_random_selection_golden(M):
    from paper_2504_06067_b200 import errors
    offs, cand = np.array([0, 3]), np.array([7, 4, 9])
    taken, it = M.niche.batched_random_selection(offs, cand, np.array([1]), np.array([3]), 0, np.array([0]))
    assert len(taken) == 0 and it == 0                                 # k = 0 -> unchanged
    taken, it = M.niche.batched_random_selection(offs, cand, np.array([1]), np.array([3]), 2, np.array([0]))
    assert np_(taken).tolist() == [7, 4] and it == 2                   # first 2 cursor entries
    with pytest.raises(errors.InfeasibleSplitError):
        M.niche.batched_random_selection(offs, cand, np.array([1]), np.array([3]), 4, np.array([0]))


def _random_niche_instance(rs, t):
    R, w = int(rs.integers(4, 3000)), int(rs.integers(1, 400))
    l = int(rs.integers(0, 3))
    ranks = rs.integers(0, l + 2, R).astype(np.int64)
    ranks[rs.random(R) < 0.1] = Od.DROPPED
    pi = rs.integers(0, w, R).astype(np.int64)
    d = (rs.integers(0, 6, R) / 4).astype(np.float32)                # ties in d
    pos_pop = Orng.positions(R, t, 1, Orng.STREAM_POP_SHUFFLE)
    pos_ref = Orng.positions(w, t, 1, Orng.STREAM_REF_SHUFFLE)
    return R, w, l, ranks, pi, d, pos_pop, pos_ref


def test_niche_pipeline_random_vs_oracle(M):
    """niche_counts -> nearest_selection -> build_cache -> batched_random_selection: every array and
    its order equal to the oracle's loop, on 60 random instances (ties, dropped rows, l = 0..2)."""
    rs = np.random.default_rng(7)
    for t in range(60):
        R, w, l, ranks, pi, d, pos_pop, pos_ref = _random_niche_instance(rs, t)
        rho, rho_p = On.niche_counts(pi, ranks, l, w)
        grho, grho_p = M.niche.niche_counts(pi, ranks, l, w)
        assert np.array_equal(np_(grho), rho) and np.array_equal(np_(grho_p), rho_p)
        fl = int((ranks == l).sum())
        k = int(rs.integers(0, max(1, fl)))
        near, rho2, rho_p2 = On.nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
        gnear, grho2, grho_p2 = M.niche.nearest_selection(pi, d, ranks, l, grho, grho_p, k, pos_pop, pos_ref)
        assert np.array_equal(np_(gnear), near), t
        assert np.array_equal(np_(grho2), rho2) and np.array_equal(np_(grho_p2), rho_p2)
        offs, cand = On.build_cache(pi, ranks, l, w, pos_pop, near)
        goffs, gcand = M.niche.build_cache(pi, ranks, l, w, pos_pop, near)
        assert np.array_equal(np_(goffs), offs) and np.array_equal(np_(gcand), cand)
        k_rem = k - len(near)
        if k_rem > int(rho_p2[rho2 < INF].sum()):
            continue
        taken, it = On.batched_random_selection(offs, cand, rho2, rho_p2, k_rem, pos_ref)
        gtaken, git = M.niche.batched_random_selection(goffs, gcand, grho2, grho_p2, k_rem, pos_ref)
        assert np.array_equal(np_(gtaken), taken), t
        assert git == it


# ----------------------------------------------------------------- variation

@pytest.mark.parametrize("ex", examples({"sbx_pair", "sbx_sum", "pm", "pm_lower"}), ids=lambda e: e["line"])
def test_variation_golden(M, ex):
    op = ex["op"]
    if op == "sbx_pair":
        c1, c2 = M.variation.sbx_pair(ex["p1"], ex["p2"], u=ex["u"], eta=ex["eta"])
        assert np.allclose(np_(c1), ex["c1"], atol=1e-12) and np.allclose(np_(c2), ex["c2"], atol=1e-12)
    elif op == "sbx_sum":
        c1, c2 = M.variation.sbx_pair(ex["p1"], ex["p2"], u=ex["u"], eta=ex["eta"], clamp=False)
        assert np.allclose(np_(c1) + np_(c2), np.add(ex["p1"], ex["p2"]), atol=1e-9)
    elif op == "pm":
        out = M.variation.polynomial_mutation(ex["x"], u=ex["u"], eta=ex["eta"])
        assert np.allclose(np_(out), ex["out"], atol=1e-12)
    else:
        out = M.variation.polynomial_mutation(ex["x"], u=ex["u"], eta=ex["eta"])
        assert (np_(out) >= 0.0).all()


def test_variation_random_vs_oracle(M):
    rs = np.random.default_rng(3)
    P1, P2 = rs.random((500, 9)), rs.random((500, 9))
    U = rs.random((500, 9))
    c1, c2 = M.variation.sbx_pair(P1, P2, u=U, eta=15.0, lo=0.1, hi=0.9)
    o1, o2 = Ov.sbx_pair(P1, P2, U, 15.0, 0.1, 0.9)
    assert np.allclose(np_(c1), o1, rtol=1e-12, atol=1e-14) and np.allclose(np_(c2), o2, rtol=1e-12, atol=1e-14)
    X = rs.random((300, 7))
    flag = rs.random((300, 7)) < 0.5
    out = M.variation.polynomial_mutation(X, u=U[:300, :7], eta=25.0, flag=flag, lo=-1.0, hi=2.0)
    want = np.where(flag, np.clip(Ov.pm_delta(X, U[:300, :7], 25.0, -1.0, 2.0), -1.0, 2.0), X)
    assert np.allclose(np_(out), want, rtol=1e-12, atol=1e-14)


def test_variation_engine_draws_reproduce_vary_eval(M):
    """mating_pool + sbx_pair(engine draws) + round + polynomial_mutation(engine draws) = the fused
    k_vary_eval offspring (rows 2q, 2q+1 of pair q)."""
    n, d, seed, gen = 200, 11, 5, 3
    X = np.random.default_rng(0).random((n, d)).astype(np.float32)
    cfg = M.variation.VariationConfig()
    prob = M.problems.ContinuousProblem("DTLZ2", 3, d)
    Xo, _ = M.variation.vary_eval(prob, torch.from_numpy(X).cuda(), cfg, seed, gen)
    pairs = np_(M.variation.mating_pool(n, seed, gen)).astype(np.int64)
    c1, c2 = M.variation.sbx_pair(X[pairs[:, 0]].astype(np.float64), X[pairs[:, 1]].astype(np.float64), cfg=cfg,
                                  seed=seed, generation=gen)
    O = np.empty((n, d))
    O[0::2], O[1::2] = np_(c1), np_(c2)
    O32 = O.astype(np.float32).astype(np.float64)               # the engine rounds once after SBX
    out = M.variation.polynomial_mutation(O32, cfg=cfg, seed=seed, generation=gen)
    assert np.array_equal(np_(out).astype(np.float32), np_(Xo))
