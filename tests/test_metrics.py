"""metrics and the DTLZ front samplers.

CPU: the oracle's igd / exact hv against the SPEC examples; the front
samplers' analytic properties.  GPU: mo_igd against the FP64 brute force
(1e-12), its symmetry / scale equivariance, and mo_hv_mc
against the exact hypervolume within 3 standard errors;
mo_hv_exact (m <= 3) against the oracle's sweep on random / tied /
out-of-box fronts, the SPEC examples, and normalized_hv."""
import numpy as np
import pytest

from oracle.manyobj_ref import metrics as Om
from paper_2504_06067_b200 import errors


def test_oracle_igd_examples():
    Z = np.random.default_rng(0).random((20, 3))
    assert Om.igd(Z, Z) == 0.0
    assert Om.igd([[3.0, 4.0]], [[0.0, 0.0]]) == pytest.approx(5.0, abs=1e-15)
    with pytest.raises(errors.EmptySelectionError):
        Om.igd(np.zeros((0, 2)), [[0.0, 0.0]])


def test_oracle_hv_examples():
    assert Om.hv([[0.5, 0.5]], [1, 1]) == pytest.approx(0.25)
    assert Om.hv([[0.25, 0.75], [0.75, 0.25]], [1, 1]) == pytest.approx(0.3125)
    assert Om.hv([[1.0, 1.0]], [1, 1]) == 0.0
    assert Om.hv([[0.5, 0.5, 0.5]], [1, 1, 1]) == pytest.approx(0.125)
    # monotone: adding a point never decreases hv
    rs = np.random.default_rng(2)
    P = rs.random((30, 3))
    assert Om.hv(np.vstack([P, rs.random((1, 3))]), [1, 1, 1]) >= Om.hv(P, [1, 1, 1]) - 1e-15


def test_oracle_normalized_hv_examples():
    # single front {(0,0),(1,1)} -> ref (1.01,1.01), ideal (0,0), HV_max = 1.0201 -> 1.0
    assert Om.normalized_hv([[[0.0, 0.0], [1.0, 1.0]]]) == pytest.approx([1.0], rel=1e-12)
    a = [[0.2, 0.7], [0.6, 0.3]]
    v = Om.normalized_hv([a, a])
    assert v[0] == v[1] and 0.0 <= v[0] <= 1.0
    assert Om.normalized_hv([[[1.0, 0.0]], [[1.0, 0.0]]]) == [0.0, 0.0]      # HV_max = 0


def test_pf_samples_on_front():
    from paper_2504_06067_b200.metrics import dtlz_pf_sample
    for m in (2, 3, 5, 8):
        f = dtlz_pf_sample("DTLZ2", m, 500)
        assert f.shape == (500, m) and np.allclose((f ** 2).sum(1), 1.0, atol=1e-12)
        f = dtlz_pf_sample("DTLZ1", m, 300)
        assert np.allclose(f.sum(1), 0.5, atol=1e-12) and (f >= 0).all()
        f = dtlz_pf_sample("DTLZ5", m, 200)
        assert np.allclose((f ** 2).sum(1), 1.0, atol=1e-12)
        if m > 2:   # degenerate curve: f_1..f_{m-1} share one profile (theta_i = pi/4 for i >= 2)
            assert np.linalg.matrix_rank(f - f.mean(0), tol=1e-9) <= 2
    f = dtlz_pf_sample("DTLZ7", 3, 400)
    assert f.shape == (400, 3)
    keep = (f[:, None, :] <= f[None]).all(-1) & (f[:, None, :] < f[None]).any(-1)
    assert not keep.any()                                    # mutually non-dominated
    assert np.allclose(f[:, 2], 2 * 3 - (f[:, :2] * (1 + np.sin(3 * np.pi * f[:, :2]))).sum(1))
    one = dtlz_pf_sample("DTLZ2", 3, 1)
    assert one.shape == (1, 3) and np.isclose((one ** 2).sum(), 1.0)
    assert np.array_equal(dtlz_pf_sample("DTLZ3", 4, 50), dtlz_pf_sample("DTLZ3", 4, 50))
    with pytest.raises(errors.ParameterError):
        dtlz_pf_sample("MNK", 3, 10)


@pytest.mark.gpu
def test_gpu_igd_matches_brute_force():
    from paper_2504_06067_b200 import metrics
    rs = np.random.default_rng(1)
    for nf, nr, m in [(20, 20, 3), (1, 1, 2), (1000, 777, 5), (4097, 513, 10), (3, 2000, 3)]:
        F = rs.random((nf, m)).astype(np.float32)
        Z = rs.random((nr, m)).astype(np.float32)
        want = Om.igd(F.astype(np.float64), Z.astype(np.float64))
        got = metrics.igd(F, Z)
        assert got == pytest.approx(want, rel=1e-12, abs=1e-15)
        # permutation symmetry and scale equivariance (power-of-two scale: exact in FP32)
        assert metrics.igd(F[rs.permutation(nf)], Z[rs.permutation(nr)]) == pytest.approx(got, rel=1e-12)
        assert metrics.igd(F * 4, Z * 4) == pytest.approx(4 * got, rel=1e-12)
    assert metrics.igd([[3.0, 4.0]], [[0.0, 0.0]]) == 5.0
    with pytest.raises(errors.EmptySelectionError):
        metrics.igd(np.zeros((0, 2), np.float32), [[0.0, 0.0]])


@pytest.mark.gpu
def test_gpu_hv_mc_agrees_with_exact():
    from paper_2504_06067_b200 import metrics
    rs = np.random.default_rng(4)
    for trial in range(20):
        m = 2 + trial % 2
        P = rs.random((40, m)).astype(np.float32)
        P = P / np.linalg.norm(P, axis=1, keepdims=True)          # a curved front
        ref = np.full(m, 1.1)
        exact = Om.hv(P.astype(np.float64), ref)
        lo = np.zeros(m)
        est, se = metrics.hv_mc(P, ref, samples=200_000, seed=trial, lower=lo)
        assert abs(est - exact) <= 3 * se + 1e-9, (trial, est, exact, se)
    est, se = metrics.hv_mc([[0.5, 0.5]], [1, 1], samples=100_000, lower=[0, 0])
    assert abs(est - 0.25) <= 3 * se
    assert metrics.hv_mc([[2.0, 2.0]], [1, 1]) == (0.0, 0.0)


@pytest.mark.gpu
def test_gpu_hv_exact_matches_sweep():
    from paper_2504_06067_b200 import metrics
    assert metrics.hv([[0.5, 0.5]], [1, 1]) == 0.25
    assert metrics.hv([[0.25, 0.75], [0.75, 0.25]], [1, 1]) == 0.3125
    assert metrics.hv([[1.0, 1.0]], [1, 1]) == 0.0
    assert metrics.hv([[2.0, 0.0]], [1, 1]) == 0.0                       # discarded -> empty -> 0
    assert metrics.hv(np.zeros((0, 3), np.float32), [1, 1, 1]) == 0.0
    assert metrics.hv([[0.25]], [1.0]) == 0.75
    rs = np.random.default_rng(6)
    for trial, (n, m) in enumerate([(1, 3), (2, 2), (50, 3), (300, 3), (257, 2), (1000, 3), (40, 1), (3000, 3)]):
        P = rs.random((n, m)).astype(np.float32)
        if trial % 2:
            P = np.round(P * 8) / 8                                       # ties in every coordinate
            P = np.vstack([P, P[: n // 3]])                               # duplicate rows
        ref = np.full(m, 0.9)                                             # some rows fall outside
        want = Om.hv(P.astype(np.float64), ref)
        got = metrics.hv(P, ref)
        assert got == pytest.approx(want, rel=1e-12, abs=1e-15), (n, m, got, want)
        assert metrics.hv(P[rs.permutation(P.shape[0])], ref) == pytest.approx(got, rel=1e-12)
        assert metrics.hv(P, ref) == got                                  # deterministic
    # monotone: adding a point never decreases the exact hv
    P = rs.random((200, 3)).astype(np.float32)
    assert metrics.hv(np.vstack([P, rs.random((1, 3)).astype(np.float32)]), [1, 1, 1]) >= metrics.hv(P, [1, 1, 1])
    # the slab sweep at population scale (n = 20k) against the MC estimate
    P = rs.random((20_000, 3)).astype(np.float32)
    P = P / np.linalg.norm(P, axis=1, keepdims=True)
    ex = metrics.hv(P, [1.1, 1.1, 1.1])
    est, se = metrics.hv_mc(P, [1.1, 1.1, 1.1], samples=400_000, lower=[0, 0, 0])
    assert abs(est - ex) <= 4 * se


@pytest.mark.gpu
def test_gpu_normalized_hv():
    from paper_2504_06067_b200 import metrics
    assert metrics.normalized_hv([[[0.0, 0.0], [1.0, 1.0]]]) == pytest.approx([1.0], rel=1e-12)
    rs = np.random.default_rng(8)
    fronts = [rs.random((60, 3)).astype(np.float32) + 0.1 * i for i in range(3)]
    got = metrics.normalized_hv(fronts)
    want = Om.normalized_hv([f.astype(np.float64) for f in fronts])
    assert got == pytest.approx(want, rel=1e-12)
    assert all(0.0 <= v <= 1.0 for v in got)
    # dividing by (ref - ideal) and recomputing in the unit box reproduces the value
    allf = np.concatenate(fronts).astype(np.float64)
    ref, ideal = 1.01 * allf.max(0), 0.9 * allf.min(0)
    scaled = ((fronts[0] - ideal) / (ref - ideal)).astype(np.float64)
    assert Om.hv(scaled, np.ones(3)) == pytest.approx(got[0], abs=1e-6)   # FP32 front, FP64 box
    with pytest.warns(RuntimeWarning):
        assert metrics.normalized_hv([[[1.0, 0.0]], [[1.0, 0.0]]]) == [0.0, 0.0]
    # m > 3: the Monte-Carlo branch, fixed seed -> reproducible
    f5 = [rs.random((100, 5)).astype(np.float32)]
    assert metrics.normalized_hv(f5, samples=200_000) == metrics.normalized_hv(f5, samples=200_000)
