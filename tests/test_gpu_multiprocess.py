"""Real multi-process sharded generations on the GPU: G processes (one per
shard, all on cuda:0 here -- this box has one GPU) run Engine(group=...) with
the production host protocol (Engine.step_gen + run_collective; gloo with
host-staged buffers instead of NCCL) and real kernels.  Every rank must hold
exactly the single-process survivors after every generation."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {"dtlz7": dict(problem="DTLZ7", n=3000, m=3, d=22), "dtlz2m6": dict(problem="DTLZ2", n=2000, m=6, d=15)}


def _worker(rank, world, port, case, gens, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2504_06067_b200 import engine
        cfg = engine.RunConfig(generations=gens, seed=5, **CASES[case])
        eng = engine.Engine(cfg, group=dist.group.WORLD)
        assert eng.host_fronts and eng.shard_count == world
        snaps = []
        for _ in range(gens):
            eng.step()
            snaps.append(torch.cat([eng.X.flatten(), eng.F.flatten()]).cpu())
        torch.save(snaps, f"{out}.{rank}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "dtlz7"), (3, "dtlz2m6")])
def test_multiprocess_shards_equal_single_gpu(tmp_path, world, case):
    gens = 3
    out = str(tmp_path / "snap")
    mp.spawn(_worker, args=(world, _free_port(), case, gens, out), nprocs=world)
    from paper_2504_06067_b200 import engine
    cfg = engine.RunConfig(generations=gens, seed=5, **CASES[case])
    one = engine.Engine(cfg, sort="stream")
    want = []
    for _ in range(gens):
        one.step()
        want.append(torch.cat([one.X.flatten(), one.F.flatten()]).cpu())
    for r in range(world):
        got = torch.load(f"{out}.{r}")
        for g in range(gens):
            assert torch.equal(got[g], want[g]), (r, g)
