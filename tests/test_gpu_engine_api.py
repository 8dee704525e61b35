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
