"""Engine host API on the GPU: device-side errors are raised with the reference's exception classes
(errors.py:4-41), and graph replays stay in step with eager generations."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import paper_2504_06067_b200 as pkg
    from paper_2504_06067_b200 import _lib
    _lib.lib()
    return pkg


def test_device_status_raises_mapped_error(M):
    from paper_2504_06067_b200 import _lib, errors
    eng = M.engine.Engine(M.engine.RunConfig(problem="DTLZ1", n=92, m=3, d=7, seed=1))
    eng.step()
    eng.check_errors()                                   # clean run: nothing raised
    eng.info[_lib.INFO["ERROR_FIRST"]] = 6               # as k_front_peel / k_stream_mark write it
    with pytest.raises(errors.InfeasibleSplitError):
        eng.check_errors()
    eng.check_errors()                                   # raised once, then cleared
    # lazily, one step late, without an explicit check
    eng.info[_lib.INFO["ERROR_FIRST"]] = 6
    eng.step()
    torch.cuda.synchronize()
    with pytest.raises(errors.InfeasibleSplitError):
        eng.step()


def test_run_raises_at_end(M):
    from paper_2504_06067_b200 import _lib, errors
    cfg = M.engine.RunConfig(problem="DTLZ2", n=100, m=3, d=12, generations=2, seed=2)
    eng = M.engine.Engine(cfg, graph=True)
    eng.info[_lib.INFO["ERROR_FIRST"]] = 5
    with pytest.raises(errors.DomainError):
        eng.replay(2)


def test_replay_after_eager_steps(M):
    """replay_one after eager steps reads the right device generation (the RNG streams depend on it)."""
    cfg = M.engine.RunConfig(problem="DTLZ2", n=200, m=4, d=13, generations=6, seed=8)
    a = M.engine.Engine(cfg, graph=True)
    a.step()
    a.step()
    a.replay_one()
    a.step()
    a.replay_one()
    b = M.engine.Engine(cfg)
    for _ in range(5):
        b.step()
    torch.cuda.synchronize()
    assert a.generation == b.generation == 5
    assert torch.equal(a.X, b.X) and torch.equal(a.F, b.F) and torch.equal(a.ideal, b.ideal)


def test_snapshot_resume_bit_identical(tmp_path):
    """SPEC.md:437 / :492 run-state snapshots: a run resumed from a snapshot continues bit-identically
    (the RNG streams are keyed by (seed, generation))."""
    import torch

    from paper_2504_06067_b200 import engine
    cfg = engine.RunConfig(problem="DTLZ2", n=600, m=5, d=14, generations=10, seed=3)
    a = engine.initialize(cfg)
    for _ in range(10):
        a = engine.step(a)
    b = engine.initialize(cfg)
    for _ in range(5):
        b = engine.step(b)
    path = str(tmp_path / "snap.npz")
    engine.save_state(b, path)
    c = engine.load_state(path)
    assert c.generation == 5
    for _ in range(5):
        c = engine.step(c)
    torch.cuda.synchronize()
    assert c.generation == a.generation == 10
    assert torch.equal(c.X, a.X) and torch.equal(c.F, a.F) and torch.equal(c.ideal, a.ideal)
    other = engine.RunConfig(problem="DTLZ2", n=600, m=5, d=14, generations=10, seed=4)
    with pytest.raises(Exception):
        engine.load_state(path, cfg=other)


@pytest.mark.parametrize("kind,n,m,d,gens", [("DTLZ2", 2000, 5, 14, 4), ("DTLZ1", 92, 3, 7, 6),
                                             ("DTLZ3", 3000, 10, 19, 3), ("DTLZ7", 1500, 3, 22, 4)])
def test_debug_bookkeeping_every_generation(kind, n, m, d, gens):
    """SPEC.md:406 debug mode: after every generation the niche counts, nearest promotions, takes, water
    level and cache order recomputed from scratch agree with the kernels' state; the trace has one
    record per generation."""
    from paper_2504_06067_b200 import engine, niche
    cfg = engine.RunConfig(problem=kind, n=n, m=m, d=d, generations=gens, seed=7)
    eng = engine.Engine(cfg, debug=True)
    niched = 0
    for _ in range(gens):
        eng.step()                   # raises on any inconsistency
        niched += 1 - eng.info_dict()["skipped"]
    assert len(eng.niche_trace) == gens and niched > 0
    rep = niche.check_bookkeeping(eng)
    assert all(rep.values()), rep
    # the checker is not vacuous: a corrupted take is detected
    st = niche.niche_state(eng)
    if not eng.info_dict()["skipped"] and int(st["take"].sum()) > 0:
        j = int(torch_nonzero_first(st["take"]))
        st["take"][j] += 1
        assert not all(niche.check_bookkeeping(eng).values())


def torch_nonzero_first(t):
    import torch
    return torch.nonzero(t).flatten()[0]
