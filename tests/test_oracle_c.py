"""The C/OpenMP restatement (oracle/c, bench.py's "fair multi-core" CPU baseline) against the numpy
oracle it restates: non_dominated_sort ranks (with and without stop_at) and the canonical FP32
association, bit for bit, on random, tied and duplicated rows.  CPU only."""
import numpy as np
import pytest

from oracle import c as oc
from oracle.manyobj_ref import dominance as Od
from oracle.manyobj_ref import niche as On
from oracle.manyobj_ref import refpoints as Oref
from oracle.manyobj_ref import rng as Orng


@pytest.mark.parametrize("R,m", [(1, 3), (2, 2), (50, 2), (300, 3), (777, 5), (500, 10), (130, 16)])
def test_c_nds_matches_oracle(R, m):
    rs = np.random.default_rng(R * 31 + m)
    for tie in (False, True):
        F = rs.random((R, m)).astype(np.float32)
        if tie:
            F = (np.round(F * 5) / 5).astype(np.float32)
            F[: R // 4] = F[R // 4: 2 * (R // 4)]                   # duplicated rows
        for stop in (None, max(1, R // 2), R):
            assert np.array_equal(oc.nds(F, stop), Od.non_dominated_sort(F, stop_at=stop)), (R, m, tie, stop)
        rows = np.arange(0, R, 3)
        D = Od.dominance_matrix(F)
        assert np.array_equal(oc.dominator_counts(F, rows=rows), D.sum(axis=0)[rows])


@pytest.mark.parametrize("m,n", [(2, 30), (3, 92), (5, 1000), (8, 300), (10, 200)])
def test_c_associate_bit_exact(m, n):
    rs = np.random.default_rng(m)
    zh = Oref.unit_directions(Oref.reference_points(m, n)).astype(np.float32)
    w = zh.shape[0]
    pos = Orng.positions(w, 3, 1, Orng.STREAM_REF_SHUFFLE)
    Fn = rs.random((900, m)).astype(np.float32)
    Fn[:100] = np.round(Fn[:100] * 4) / 4                          # ties between references
    Fn[100] = 0.0                                                  # the origin: all dots 0 -> first by position
    p1, d1 = On.associate_canonical(Fn, zh, pos, np.arange(900))
    p2, d2 = oc.associate(Fn, zh, pos)
    assert np.array_equal(p1, p2)
    assert np.array_equal(d1.view(np.int32), d2.view(np.int32))
    rows = np.array([5, 100, 899])
    p3, d3 = oc.associate(Fn, zh, pos, rows=rows, threads=2)
    assert np.array_equal(p3, p1[rows]) and np.array_equal(d3, d1[rows])
