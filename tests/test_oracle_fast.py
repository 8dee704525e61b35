"""The accelerated checker used by the BASELINE-size parity tests (tests/test_gpu_baseline_sizes.py)
against the plain numpy oracle it stands in for.  CPU only.

* oracle/c nds3 (lexicographic staircase sweep, m <= 3) == the peeling NDS of
  oracle/manyobj_ref/dominance.py:36, with and without stop_at, on random,
  tied, duplicated and signed-zero rows;
* niche.nearest_selection_vec == niche.nearest_selection;
* a whole survivor selection with oracle/c's accel() == the numpy selection, generation after
  generation of a real run (the same survivors, ranks, pi, d).
"""
import numpy as np
import pytest

from oracle import c as oc
from oracle.manyobj_ref import dominance as Od
from oracle.manyobj_ref import engine as Oeng
from oracle.manyobj_ref import niche as On
from oracle.manyobj_ref import rng as Orng


def _instances(rs, count):
    for t in range(count):
        R = int(rs.integers(1, 400))
        m = int(rs.integers(1, 4))
        kind = t % 4
        if kind == 0:
            F = rs.random((R, m)).astype(np.float32)
        elif kind == 1:
            F = rs.integers(0, 4, (R, m)).astype(np.float32)          # many ties
        elif kind == 2:
            F = rs.integers(-1, 2, (R, m)).astype(np.float32)
            F[rs.random((R, m)) < 0.4] *= -0.0                      # -0 vs +0
        else:
            F = rs.random((R, m)).astype(np.float32)
            F[R // 2:] = F[: R - R // 2]                              # duplicated rows
        yield F


def test_nds3_matches_peeling_oracle():
    rs = np.random.default_rng(5)
    for F in _instances(rs, 240):
        R = F.shape[0]
        for stop in (None, int(rs.integers(1, R + 1)), R):
            want = Od.non_dominated_sort(F, stop_at=stop)
            assert np.array_equal(oc.nds3(F, stop), want), (F.shape, stop)


def test_nds3_chain_and_antichain():
    chain = np.stack([np.arange(500, dtype=np.float32)] * 3, axis=1)
    assert np.array_equal(oc.nds3(chain), np.arange(500))
    t = np.linspace(0, 1, 400, dtype=np.float32)
    anti = np.stack([t, 1 - t, np.zeros_like(t)], axis=1)
    assert (oc.nds3(anti) == 0).all()


def test_nds_auto_dispatch():
    rs = np.random.default_rng(1)
    F = rs.random((300, 5)).astype(np.float32)
    assert np.array_equal(oc.nds_auto(F, 150), Od.non_dominated_sort(F, stop_at=150))


def test_nearest_selection_vec_equals_loop():
    rs = np.random.default_rng(11)
    for t in range(200):
        R, w = int(rs.integers(4, 120)), int(rs.integers(1, 20))
        l = int(rs.integers(0, 3))
        ranks = rs.integers(0, l + 2, R).astype(np.int64)
        ranks[rs.random(R) < 0.1] = Od.DROPPED
        pi = rs.integers(0, w, R).astype(np.int64)
        d = (rs.integers(0, 4, R) / 4).astype(np.float32)          # ties in d
        pos_pop = Orng.positions(R, t, 0, Orng.STREAM_POP_SHUFFLE)
        pos_ref = Orng.positions(w, t, 0, Orng.STREAM_REF_SHUFFLE)
        rho, rho_p = On.niche_counts(pi, ranks, l, w)
        k = int(rs.integers(0, 8))
        a = On.nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
        b = On.nearest_selection_vec(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ1", 92, 3, 7, 12), ("DTLZ2", 300, 5, 14, 6),
                                             ("DTLZ3", 200, 10, 19, 4), ("DTLZ7", 400, 3, 22, 6)])
def test_accelerated_selection_equals_numpy(kind, n, m, d, gens):
    cfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=3)
    st_a = Oeng.initialize(cfg)
    st_b = Oeng.initialize(cfg)
    acc = oc.accel(threads=2)
    for _ in range(gens):
        st_a = Oeng.step(st_a, cfg)
        st_b = Oeng.step(st_b, cfg, **acc)
        assert np.array_equal(st_a.X, st_b.X) and np.array_equal(st_a.F, st_b.F)
        assert np.array_equal(st_a.info["ranks"], st_b.info["ranks"])
        assert st_a.info["l"] == st_b.info["l"] and st_a.info["k"] == st_b.info["k"]
        if not st_a.info["skipped"]:
            assert np.array_equal(st_a.info["pi"], st_b.info["pi"])
            assert np.array_equal(st_a.info["d"].view(np.int32), st_b.info["d"].view(np.int32))
