"""Streamed / sharded non-dominated sort and sharded association (GPU).

The streamed sort (mo_sort_stream_*: dominator counts + per-front
count-decrement, no bit-matrix) must give the oracle's ranks and split on
the same objectives, for 1..8 shards exchanging their front masks; an engine
in streamed mode must produce bit-identical generations to the bit-matrix
engine; and G shards (emulated in one process on one GPU: every shard has its
own workspace and only sees its shard index; the collectives are the same
bytes NCCL moves) must produce bit-identical generations to one GPU.
"""
import numpy as np
import pytest
import torch

from oracle.manyobj_ref import dominance as Odom

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2504_06067_b200 as pkg
    from paper_2504_06067_b200 import _lib
    _lib.lib()
    return pkg


def np_(t):
    return t.detach().cpu().numpy()


def _cases():
    rs = np.random.default_rng(31)
    for R, m in [(4, 2), (64, 3), (184, 3), (512, 2), (772, 5), (1000, 10), (2048, 3), (3000, 4), (600, 12), (900, 16)]:
        yield rs.random((R, m)).astype(np.float32)
        yield rs.integers(0, 4, size=(R, m)).astype(np.float32)           # ties + duplicates
    x = np.sort(rs.random(600)).astype(np.float32)
    yield np.stack([x, x, x], 1)                                          # one chain: 600 fronts
    yield np.repeat(rs.random((100, 3)).astype(np.float32), 4, axis=0)    # every row 4 times
    yield np.zeros((256, 5), np.float32)                                  # all identical
    x = rs.random(2000).astype(np.float32)
    yield np.stack([x, 1 - x], 1).astype(np.float32)                       # all mutually non-dominated


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_stream_sort_matches_oracle(M, shards):
    for F in _cases():
        R = F.shape[0]
        n = R // 2
        ranks, info = M.dominance.stream_sort(F, n, shards=shards, poll=1 + (R % 3))
        want = Odom.non_dominated_sort(F, stop_at=n)
        assert np.array_equal(np_(ranks), want), (F.shape, shards)
        sp = M.dominance.split_from_info(info)
        wsp = Odom.split_fronts(want, n)
        assert (sp.l, sp.selected_count, sp.k) == (wsp.l, wsp.selected_count, wsp.k), (F.shape, shards)
        h = np_(info)
        assert h[M._lib.INFO["NFRONTS"]] == wsp.l + 1


def test_stream_sort_equals_bits_path_large(M):
    """R = 40,000 (m = 3, random + ties): streamed ranks == the bit-matrix peel's ranks."""
    rs = np.random.default_rng(5)
    for F in (rs.random((40000, 3)).astype(np.float32),
              (rs.integers(0, 50, size=(40000, 3)) / 50).astype(np.float32)):
        n = 20000
        r1, i1 = M.dominance.stream_sort(F, n, shards=1, poll=4)
        r2, i2 = M.dominance.non_dominated_sort(F, stop_at=n, return_info=True)
        assert torch.equal(r1, r2)
        for key in ("L", "SELECTED", "K", "NFRONTS", "FL_SIZE", "SKIPPED"):
            assert int(i1[M._lib.INFO[key]]) == int(i2[M._lib.INFO[key]]), key
        r3, _ = M.dominance.stream_sort(F, n, shards=4, poll=4)
        assert torch.equal(r1, r3)


@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ2", 1000, 5, 14, 5), ("DTLZ7", 2000, 3, 22, 5),
                                             ("DTLZ3", 600, 10, 19, 4), ("DTLZ1", 92, 3, 7, 20)])
def test_stream_engine_equals_bits_engine(M, kind, n, m, d, gens):
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=3)
    a = M.engine.Engine(cfg, sort="bits")
    b = M.engine.Engine(cfg, sort="stream", host_fronts=False)   # device-side front loop (k_stream_fused)
    c = M.engine.Engine(cfg, sort="stream", host_fronts=True)    # host-driven fronts (the sharded protocol)
    assert not b.host_fronts and c.host_fronts
    for g in range(gens):
        a.step()
        b.step()
        c.step()
        for e in (b, c):
            assert torch.equal(a.X, e.X) and torch.equal(a.F, e.F), f"generation {g}"
            assert torch.equal(a.ideal, e.ideal)
            assert a.info_dict() == e.info_dict()


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_local_shards_equal_one_gpu(M, shards):
    cfg = M.engine.RunConfig(problem="DTLZ7", n=1500, m=3, d=22, generations=4, seed=11)
    one = M.engine.Engine(cfg, sort="stream")
    grp = M.engine.LocalShards(cfg, shards)
    for g in range(4):
        one.step()
        grp.step()
        for e in grp.engines:
            assert torch.equal(e.X, one.X) and torch.equal(e.F, one.F), (shards, g)
            assert torch.equal(e.ideal, one.ideal)
            assert e.info_dict() == one.info_dict()


def test_local_shards_m10(M):
    cfg = M.engine.RunConfig(problem="DTLZ3", n=800, m=10, d=19, generations=3, seed=2)
    one = M.engine.Engine(cfg, sort="bits")
    grp = M.engine.LocalShards(cfg, 3)
    for _ in range(3):
        one.step()
        grp.step()
        for e in grp.engines:
            assert torch.equal(e.X, one.X) and torch.equal(e.F, one.F)


def test_stream_engine_profile_and_poll(M):
    cfg = M.engine.RunConfig(problem="DTLZ7", n=3000, m=3, d=22, generations=3, seed=1)
    a = M.engine.Engine(cfg, sort="stream", poll=1, host_fronts=True)
    b = M.engine.Engine(cfg, sort="stream", poll=16, host_fronts=True)
    prof = {}
    for _ in range(3):
        a.step(profile=prof)
        b.step()
    assert torch.equal(a.X, b.X)
    assert prof["t_sort"] > 0 and prof["fronts_issued"] >= 1


# ------------------------------------------------------- lattice-pruned association

@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ7", 3000, 3, 22, 6), ("DTLZ1", 2000, 3, 7, 6),
                                             ("DTLZ2", 4000, 4, 13, 5), ("DTLZ5", 1000, 2, 11, 5),
                                             ("DTLZ4", 5000, 3, 12, 5), ("DTLZ2", 10000, 5, 14, 4),
                                             ("DTLZ1", 6000, 5, 9, 4)])
def test_lattice_pruned_association_equals_full_scan(M, kind, n, m, d, gens):
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=6)
    a = M.engine.Engine(cfg, prune=False)
    b = M.engine.Engine(cfg, prune=True)
    assert a.lattice is None and b.lattice is not None
    for g in range(gens):
        a.step()
        b.step()
        assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F), (kind, g)
        ia, ib = a.info_dict(), b.info_dict()
        fb = ib.pop("assoc_fallback")
        ia.pop("assoc_fallback")
        assert ia == ib
        if not ib["skipped"]:
            assert fb < 0.02 * n, fb          # the certificate holds for almost every candidate


def test_lattice_pruned_association_adversarial(M):
    """Candidates on lattice directions, on cell boundaries, on the simplex edges and at the ideal point."""
    from paper_2504_06067_b200 import _lib
    cfg = M.engine.RunConfig(problem="DTLZ1", n=2000, m=3, d=7, generations=1, seed=2)
    rs = np.random.default_rng(3)
    n = 2000
    Z = M.refpoints.reference_points(3, n)
    H = M.refpoints.choose_divisions(3, n)[0]
    F = np.concatenate([
        Z[rs.integers(0, len(Z), 800)] * rs.uniform(0.5, 2.0, (800, 1)),           # exactly on directions
        (np.floor(rs.random((800, 3)) * H) + 0.5) / H,                            # cell midpoints
        np.eye(3)[rs.integers(0, 3, 600)] * rs.random((600, 1)),                  # simplex vertices
        np.concatenate([rs.random((600, 2)), np.zeros((600, 1))], 1),             # an edge
        np.zeros((200, 3)),                                                        # the ideal point
        rs.random((1000, 3)),
    ]).astype(np.float32)
    F = np.concatenate([np.zeros((1, 3), np.float32), F])[:2 * n]
    outs = []
    for prune in (False, True):
        eng = M.engine.Engine(cfg, prune=prune)
        eng.FR[eng.cur].copy_(torch.from_numpy(F))
        a = eng._args[eng.cur]
        L = _lib.lib()
        _lib.check(L.mo_step_phases(a, _lib.PHASE_SORT | _lib.PHASE_NICHE, _lib.stream_ptr()), "select")
        torch.cuda.synchronize()
        ao = _lib.stream_offsets(n, 3, eng.w, eng.sort_mode, 1)[3]
        akey = np_(eng.ws[ao: ao + 8 * 2 * n].view(torch.int64)).copy()
        info = eng.info_dict()
        info.pop("assoc_fallback")
        outs.append((np_(eng.FR[eng.cur ^ 1][:n]).copy(), np_(eng.ranks).copy(), info, akey))
    assert (outs[0][3] != 0).sum() > n                       # the association keys of every candidate row
    assert np.array_equal(outs[0][3], outs[1][3])
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_local_shards_with_lattice(M):
    cfg = M.engine.RunConfig(problem="DTLZ7", n=3000, m=3, d=22, generations=3, seed=8)
    one = M.engine.Engine(cfg, sort="bits", prune=False)
    grp = M.engine.LocalShards(cfg, 4, prune=True)
    for _ in range(3):
        one.step()
        grp.step()
        for e in grp.engines:
            assert torch.equal(e.X, one.X) and torch.equal(e.F, one.F)


@pytest.mark.parametrize("kind,m,n", [("DTLZ7", 3, 3000), ("DTLZ4", 3, 2000), ("DTLZ2", 6, 1500)])
def test_stream_graph_replay_equals_eager(M, kind, m, n):
    """One shard: the whole streamed generation is one mo_step, so it captures into a CUDA graph."""
    cfg = M.engine.RunConfig(problem=kind, n=n, m=m, d=m + 9, generations=6, seed=12)
    a = M.engine.Engine(cfg, sort="stream", host_fronts=False)
    for _ in range(6):
        a.step()
    b = M.engine.Engine(cfg, sort="stream", graph=True)
    b.replay(6)
    torch.cuda.synchronize()
    assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F) and a.info_dict() == b.info_dict()


def test_stream_many_fronts(M):
    """A chain-like population (hundreds of fronts) through the device-side front loop."""
    x = np.sort(np.random.default_rng(3).random(1024)).astype(np.float32)
    F = np.stack([x, x + 1, x + 2], 1)
    for stream in (True, False):
        cfg = M.engine.RunConfig(problem="DTLZ7", n=512, m=3, d=22, generations=1, seed=0)
        eng = M.engine.Engine(cfg, sort="stream" if stream else "bits")
        eng.FR[eng.cur].copy_(torch.from_numpy(F))
        from paper_2504_06067_b200 import _lib
        _lib.check(_lib.lib().mo_step_phases(eng._args[eng.cur], _lib.PHASE_SORT, _lib.stream_ptr()), "sort")
        torch.cuda.synchronize()
        r = np_(eng.ranks)
        want = Odom.non_dominated_sort(F, stop_at=512)
        assert np.array_equal(r, want), stream
        assert eng.info_dict()["nfronts"] == 512


def test_stream_auto_front_loop_switch(M):
    """Eager streamed runs switch to the device-side front loop once a generation has > 300 fronts
    (DTLZ4 m=3: hundreds); every generation still equals the bit-matrix engine."""
    cfg = M.engine.RunConfig(problem="DTLZ4", n=8000, m=3, d=12, generations=4, seed=1)
    a = M.engine.Engine(cfg, sort="bits")
    b = M.engine.Engine(cfg, sort="stream")
    switched = False
    for _ in range(4):
        switched |= b._fronts_hint > 300
        a.step()
        b.step()
        assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F)
    assert switched, b._fronts_hint
