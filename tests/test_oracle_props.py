"""Property / statistical checks of the CPU oracle (SPEC.md invariants + acceptance criteria).

These pin the oracle before the GPU is compared against it: NDS against a
textbook brute force (criterion 3), the closed-form water-fill against the
literal Alg. 2 loop, forced-choice exactness batched == Alg. 1 (criterion 2),
the loop-count bound (criterion 4), distributional equivalence batched ~ Alg.
1 (criterion 1, reduced trial count for CI), Eq. (2) geometry (criterion 10),
shuffle / mating-pool uniformity, and determinism (criterion 9).
"""
import itertools
from collections import Counter

import numpy as np
import pytest
from scipy.stats import chisquare

from oracle.manyobj_ref import batchcore, dominance, engine, niche, problems, rng, variation


def textbook_nds(F):
    """O(R^2 m * fronts) peeling straight from the definition."""
    R = len(F)
    ranks = [-1] * R
    left = set(range(R))
    k = 0
    while left:
        front = [j for j in left if not any(dominance.dominates(F[i], F[j]) for i in left if i != j)]
        for j in front:
            ranks[j] = k
        left -= set(front)
        k += 1
    return ranks


def test_nds_matches_textbook_1000():
    rs = np.random.default_rng(7)
    for t in range(1000):
        R = int(rs.integers(1, 65))
        m = int(rs.integers(1, 9))
        # few distinct values -> many ties and duplicates
        F = rs.integers(0, 4, size=(R, m)).astype(np.float64) if t % 2 else rs.random((R, m))
        assert dominance.non_dominated_sort(F).tolist() == textbook_nds(F)


def test_nds_permutation_equivariance():
    rs = np.random.default_rng(3)
    F = rs.integers(0, 5, size=(60, 3)).astype(float)
    r = dominance.non_dominated_sort(F)
    p = rs.permutation(60)
    assert np.array_equal(dominance.non_dominated_sort(F[p]), r[p])


def test_waterfill_equals_loop():
    rs = np.random.default_rng(11)
    for _ in range(4000):
        w = int(rs.integers(1, 14))
        rho = rs.integers(0, 5, size=w).astype(np.int64)
        rho_p = rs.integers(0, 5, size=w).astype(np.int64)
        rho[rho_p == 0] = niche.INF
        tot = int(rho_p[rho < niche.INF].sum())
        if tot == 0:
            continue
        k = int(rs.integers(1, tot + 1))
        pos_ref = rs.permutation(w)
        offs = np.zeros(w + 1, np.int64)
        offs[1:] = np.cumsum(rho_p)
        cand = np.arange(offs[-1])
        a, _ = niche.batched_random_selection(offs, cand, rho, rho_p, k, pos_ref)
        b = niche.waterfill_selection(offs, cand, rho, rho_p, k, pos_ref)
        assert sorted(a.tolist()) == sorted(b.tolist())


def _random_instance(rs, R, w, l_front_frac=0.5):
    """Random (pi, d, ranks, l, k) niching instance."""
    pi = rs.integers(0, w, size=R)
    d = rs.random(R).astype(np.float32)
    ranks = np.where(rs.random(R) < l_front_frac, 1, 0)
    l = 1
    n_sel = int((ranks < l).sum())
    fl = int((ranks == l).sum())
    if fl < 2:
        return None
    k = int(rs.integers(1, fl))
    return pi, d, ranks, l, k, n_sel


def test_loop_count_bound():
    rs = np.random.default_rng(5)
    fewer = total = 0
    for _ in range(100):
        w = int(rs.integers(4, 9))
        inst = _random_instance(rs, 16, w)
        if inst is None:
            continue
        pi, d, ranks, l, k, _ = inst
        rho, rho_p = niche.niche_counts(pi, ranks, l, w)
        pos_pop = rs.permutation(len(pi))
        pos_ref = rs.permutation(w)
        near, rho2, rho_p2 = niche.nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
        offs, cq = niche.build_cache(pi, ranks, l, w, pos_pop, near)
        k_rem = k - len(near)
        _, it = niche.batched_random_selection(offs, cq, rho2, rho_p2, k_rem, pos_ref)
        assert it <= k_rem
        if k_rem > 0:
            total += 1
            fewer += it < k_rem
    assert total > 0 and fewer / total >= 0.3


def _forced_instance(rs, w):
    """Every reference point has rho=0 and exactly one candidate with a unique distance, k = w."""
    pi = np.arange(w)
    d = rs.random(w).astype(np.float32)
    ranks = np.zeros(w, int)
    return pi, d, ranks, 0, w


def test_forced_choice_batched_equals_oracle_100():
    rs = np.random.default_rng(9)
    for _ in range(100):
        w = int(rs.integers(1, 7))
        pi, d, ranks, l, k = _forced_instance(rs, w)
        rho, rho_p = niche.niche_counts(pi, ranks, l, w)
        near, *_ = niche.nearest_selection(pi, d, ranks, l, rho, rho_p, k, rs.permutation(w), rs.permutation(w))
        orc = niche.oracle_niche_select(pi, d, ranks, l, k, w, np.random.default_rng(int(rs.integers(1 << 30))))
        assert sorted(near.tolist()) == sorted(orc.tolist())


def _batched_select(pi, d, ranks, l, k, w, seed):
    R = len(pi)
    pos_pop = rng.positions(R, seed, 0, rng.STREAM_POP_SHUFFLE)
    pos_ref = rng.positions(w, seed, 0, rng.STREAM_REF_SHUFFLE)
    rho, rho_p = niche.niche_counts(pi, ranks, l, w)
    near, rho2, rho_p2 = niche.nearest_selection(pi, d, ranks, l, rho, rho_p, k, pos_pop, pos_ref)
    offs, cq = niche.build_cache(pi, ranks, l, w, pos_pop, near)
    rest = niche.waterfill_selection(offs, cq, rho2, rho_p2, k - len(near), pos_ref)
    return tuple(sorted(np.concatenate([near, rest]).tolist()))


@pytest.mark.parametrize("inst_seed", range(6))
def test_batched_matches_oracle_in_distribution(inst_seed):
    """Criterion 1 on small instances (2n <= 16, w <= 6), 3000 trials each for CI speed."""
    rs = np.random.default_rng(100 + inst_seed)
    w = int(rs.integers(2, 7))
    while True:
        inst = _random_instance(rs, 12, w)
        if inst is not None:
            break
    pi, d, ranks, l, k, _ = inst
    T = 3000
    a = Counter(_batched_select(pi, d, ranks, l, k, w, s) for s in range(T))
    g = np.random.default_rng(inst_seed)
    b = Counter(tuple(sorted(niche.oracle_niche_select(pi, d, ranks, l, k, w, g).tolist())) for _ in range(T))
    keys = sorted(set(a) | set(b))
    obs = np.array([[a.get(x, 0), b.get(x, 0)] for x in keys], float)
    # two-sample chi-square homogeneity test
    from scipy.stats import chi2_contingency
    if len(keys) == 1:
        return
    p = chi2_contingency(obs.T)[1]
    assert p > 0.001, (p, keys, obs)


def test_eq2_geometry_vs_projection():
    rs = np.random.default_rng(4)
    F = rs.random((10000, 3)) * rs.random((10000, 1)) * 3
    Z = rs.random((10000, 3)) + 1e-3
    D = niche.perpendicular_distance_matrix(F[:100], Z[:100])
    for i in range(100):
        for j in range(0, 100, 7):
            z = Z[j] / np.linalg.norm(Z[j])
            proj = F[i] - np.dot(F[i], z) * z
            assert abs(D[i, j] - np.linalg.norm(proj)) < 1e-9


def test_canonical_association_agrees_with_spec_argmin():
    """argmax of the FP32 key t picks the SPEC.md argmin-D point up to FP32 near-ties."""
    rs = np.random.default_rng(8)
    Z = np.array(__import__("oracle.manyobj_ref.refpoints", fromlist=["x"]).das_dennis(3, 12))
    zh = (Z / np.linalg.norm(Z, axis=1)[:, None]).astype(np.float32)
    F = rs.random((500, 3)).astype(np.float32)
    pi_c, d_c = niche.associate_canonical(F, zh, np.arange(len(Z)), np.arange(500))
    D = niche.perpendicular_distance_matrix(F.astype(np.float64), Z)
    pi_s, d_s = niche.associate(D)
    agree = (pi_c == pi_s)
    # where they disagree the two distances are equal to FP32 precision
    assert np.allclose(D[np.arange(500), pi_c], d_s, atol=1e-6)
    assert agree.mean() > 0.99
    assert np.allclose(d_c, d_s, atol=1e-5)


def test_shuffle_uniform_3rows():
    c = Counter()
    m = batchcore.MaskedMatrix(np.arange(3.0)[:, None])
    for s in range(10000):
        _, perm = batchcore.shuffle_rows(m, batchcore.SeedableRng(s, 5))
        c[tuple(perm.tolist())] += 1
    assert len(c) == 6
    for v in c.values():
        assert abs(v / 10000 - 1 / 6) < 0.02


def test_shuffle_deterministic():
    a = rng.permutation(1000, 42, 3, rng.STREAM_POP_SHUFFLE)
    b = rng.permutation(1000, 42, 3, rng.STREAM_POP_SHUFFLE)
    assert np.array_equal(a, b) and sorted(a.tolist()) == list(range(1000))


def test_mating_pool_pairing_frequency():
    c = Counter()
    for s in range(10000):
        pairs = variation.mating_pool(4, s, 0)
        c[frozenset(frozenset(map(int, p)) for p in pairs)] += 1
    assert len(c) == 3
    for v in c.values():
        assert abs(v / 10000 - 1 / 3) < 0.03


def test_mating_pool_odd():
    from paper_2504_06067_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        variation.mating_pool(5, 0, 0)


def test_mutation_rate():
    n, d = 1000, 100
    X = np.full((n, d), 0.5, np.float32)
    cfg = variation.VariationConfig(p_c=0.0, p_m=0.05)
    O = variation.vary(X, cfg, 3, 0)
    rate = (O != 0.5).mean()
    se = np.sqrt(0.05 * 0.95 / (n * d))
    # u=0.5 exactly leaves x unchanged; probability 2^-24, negligible
    assert abs(rate - 0.05) < 3 * se


def test_variation_bounds_and_identity():
    rs = np.random.default_rng(1)
    X = rs.random((64, 9)).astype(np.float32)
    O = variation.vary(X, variation.VariationConfig(), 5, 2)
    assert (O >= 0).all() and (O <= 1).all()
    ident = variation.vary(X, variation.VariationConfig(p_c=0.0, p_m=0.0), 5, 2)
    pairs = variation.mating_pool(64, 5, 2).reshape(-1)
    assert np.array_equal(ident, X[pairs])


@pytest.mark.parametrize("kind", problems.KINDS)
def test_dtlz_batched_equals_scalar(kind):
    rs = np.random.default_rng(2)
    P = problems.ContinuousProblem(kind, 4, 9)
    X = rs.random((32, 9))
    F = problems.dtlz_eval(P, X)
    for i in range(32):
        assert np.allclose(F[i], problems.dtlz_eval(P, X[i:i + 1])[0], rtol=0, atol=0)
    assert np.isfinite(F).all() and (F >= 0).all()


def test_engine_determinism_and_size():
    cfg = engine.RunConfig(problem="DTLZ1", n=92, m=3, d=7, generations=5, seed=3)
    h1, s1 = engine.run(cfg)
    h2, s2 = engine.run(cfg)
    assert h1 == h2 and np.array_equal(s1.X, s2.X) and s1.X.shape == (92, 7)


def test_engine_identity_under_zero_variation():
    """n copies of one Pareto-optimal point + zero-probability variation -> unchanged."""
    cfg = engine.RunConfig(problem="DTLZ2", n=8, m=3, d=5, generations=1, seed=0,
                           variation=variation.VariationConfig(p_c=0.0, p_m=0.0))
    st = engine.initialize(cfg)
    x = np.array([0.3, 0.6, 0.5, 0.5, 0.5], np.float32)
    st.X = np.tile(x, (8, 1))
    st.F = engine.evaluate(cfg, st.X)
    st2 = engine.step(st, cfg)
    assert np.array_equal(st2.X, st.X)


def test_engine_batched_equals_oracle_forced():
    """on a forced instance both back-ends pick the same population."""
    cfg = engine.RunConfig(problem="DTLZ2", n=4, m=2, d=2, generations=1, seed=1)
    # four parents on the front, offspring dominated -> |F0| = 4 = n: k-skip forced
    st = engine.initialize(cfg)
    st.X = np.array([[0.1, 0.5], [0.4, 0.5], [0.6, 0.5], [0.9, 0.5]], np.float32)
    st.F = engine.evaluate(cfg, st.X)
    off = (np.full((4, 2), 0.9, np.float32), np.full((4, 2), 5.0, np.float32))
    a = engine.step(st, cfg, offspring=off)
    b = engine.step(st, engine.with_backend(cfg, "oracle"), offspring=off)
    assert np.array_equal(a.X, b.X)
