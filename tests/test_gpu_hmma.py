"""Tensor-core filtered association -- k_assoc_umma (tcgen05.mma FP16 -> FP32 in TMEM, the engine default)
and k_assoc_hmma (bf16 hi/lo m16n8k16 mma.sync) select the candidates, the canonical FP32 key decides --
against the FP32 full scan and the oracle (GPU).

* adversarial objectives -- rows on reference directions, exact midpoints between two directions (key
  ties broken by shuffled position), the ideal point (zero rows -> the sliced fallback scan), duplicates,
  huge and tiny scales -- give bit-identical association keys, ranks and survivors with and without the
  filter, at m = 3, 6, 10, 16;
* whole generations (state injection) at w >= 1024 without a lattice, m = 3 .. 16, match the oracle's
  selection exactly.
"""
import numpy as np
import pytest
import torch

from oracle.manyobj_ref import engine as Oeng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2504_06067_b200 as pkg
    from paper_2504_06067_b200 import _lib
    _lib.lib()
    return pkg


def np_(t):
    return t.detach().cpu().numpy()


def _adversarial(M, m, n, rs):
    Z = np.asarray(M.refpoints.reference_points(m, n), np.float64)
    w = len(Z)
    a = rs.integers(0, w, 600)
    b = rs.integers(0, w, 600)
    parts = [
        Z[rs.integers(0, w, 600)] * rs.uniform(0.5, 2.0, (600, 1)),          # exactly on directions
        0.5 * (Z[a] + Z[b]),                                                   # midpoints: near / exact ties
        np.zeros((50, m)),                                                     # the ideal point
        rs.random((400, m)) * 1e4,                                             # huge
        rs.random((400, m)) * 1e-4,                                            # tiny
        np.repeat(rs.random((100, m)), 3, axis=0),                             # duplicates
        rs.random((2 * n, m)),
    ]
    F = np.concatenate([np.zeros((1, m))] + parts)[:2 * n]
    return F.astype(np.float32)


def _assoc_outputs(M, eng, F, n, m):
    from paper_2504_06067_b200 import _lib
    eng.FR[eng.cur].copy_(torch.from_numpy(F))
    a = eng._args[eng.cur]
    _lib.check(_lib.lib().mo_step_phases(a, _lib.PHASE_SORT | _lib.PHASE_NICHE, _lib.stream_ptr()), "select")
    torch.cuda.synchronize()
    ao = _lib.stream_offsets(n, m, eng.w, eng.sort_mode, 1)[3]
    akey = np_(eng.ws[ao: ao + 8 * 2 * n].view(torch.int64)).copy()
    info = eng.info_dict()
    info.pop("assoc_fallback")
    return akey, np_(eng.FR[eng.cur ^ 1][:n]).copy(), np_(eng.ranks).copy(), info


@pytest.mark.parametrize("m,n", [(3, 1500), (6, 1500), (10, 1500), (16, 2000), (2, 1200), (9, 5000)])
def test_hmma_filter_bit_identical_adversarial(M, m, n):
    rs = np.random.default_rng(m)
    F = _adversarial(M, m, n, rs)
    cfg = M.engine.RunConfig(problem="DTLZ2", n=n, m=m, d=m + 9, generations=1, seed=4)
    outs = []
    for mode in ("umma", "hmma", "scan"):
        eng = M.engine.Engine(cfg, prune=False)
        assert eng.w >= 1024 and eng.zfrag is not None and eng.zumma is not None
        if mode != "umma":
            eng.zumma = None
        if mode == "scan":
            eng.zfrag = None
        eng._args = [eng._make_args(0), eng._make_args(1)]
        outs.append(_assoc_outputs(M, eng, F, n, m))
    (k1, f1, r1, i1) = outs[2]
    assert (k1 != 0).sum() > n // 2
    for k2, f2, r2, i2 in outs[:2]:
        assert np.array_equal(k1, k2)
        assert np.array_equal(f1, f2) and np.array_equal(r1, r2) and i1 == i2


def _gpu_state_to_oracle(eng):
    return Oeng.RunState(eng.generation, np_(eng.X).copy(), np_(eng.F).copy(), np_(eng.ideal).copy(),
                         M_unit(eng), np.asarray(eng.Z))


def M_unit(eng):
    from oracle.manyobj_ref import refpoints as Oref
    return Oref.unit_directions(eng.Z)


@pytest.mark.parametrize("kind,n,m,d", [("DTLZ1", 1100, 3, 7), ("DTLZ2", 1400, 5, 14), ("DTLZ3", 1100, 6, 15),
                                        ("DTLZ5", 1500, 8, 17), ("DTLZ6", 1500, 10, 19), ("DTLZ2", 2000, 16, 25)])
def test_hmma_engine_state_injection(M, kind, n, m, d):
    gens = 2
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=29)
    ocfg = Oeng.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=29)
    eng = M.engine.Engine(cfg, prune=False)
    assert eng.zfrag is not None and eng.w >= 1024
    for g in range(gens):
        st = _gpu_state_to_oracle(eng)
        cur = eng.cur
        eng.step()
        O = np_(eng.XR[cur][n:]).copy()
        FO = np_(eng.FR[cur][n:]).copy()
        nxt = Oeng.step(st, ocfg, offspring=(O, FO))
        assert np.array_equal(np_(eng.X), nxt.X), f"generation {g}"
