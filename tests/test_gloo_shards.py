"""Multi-process (world_size 2 and 3, gloo on CPU) test of the sharded
generation's host protocol: Engine.step_gen + run_collective exactly as the
NCCL path runs them, over the CPU shard emulator (tests/shard_emulator.py).
Every rank must reach the same split at the same front, the gathered ranks
must be the oracle's, and the max-reduced association keys (packed unsigned
words, sign-flipped for the signed int64 collective) must equal the
single-process full-range keys."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.manyobj_ref import dominance as Odom


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed):
    rs = np.random.default_rng(seed)
    R, m, w = 1200, 3, 91
    F = rs.random((R, m)).astype(np.float32)
    F[:300] = rs.integers(0, 4, size=(300, m)) / 4.0          # ties + duplicates
    zs = rs.random((w, m)).astype(np.float32)
    zs /= np.linalg.norm(zs, axis=1, keepdims=True)
    zs[5] = zs[17]                                               # an exact key tie across shard ranges
    return F, zs


def _worker(rank, world, port, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_06067_b200.engine import Engine, run_collective
        from shard_emulator import EmulatedShard
        F, zs = _problem(seed)
        sh = EmulatedShard(F, zs, F.shape[0] // 2, rank, world, poll=1 + seed % 3)
        for req in Engine.step_gen(sh):
            run_collective(req, dist.group.WORLD)
        res = torch.cat([torch.from_numpy(sh.ranks.astype(np.int64)), sh.finished,
                         sh.info.to(torch.int64)])
        gathered = [torch.empty_like(res) for _ in range(world)]
        dist.all_gather(gathered, res)
        if rank == 0:
            torch.save([g.clone() for g in gathered], out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 0), (3, 1), (2, 2)])
def test_gloo_sharded_generation_protocol(tmp_path, world, seed):
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(world, _free_port(), seed, out), nprocs=world)
    res = torch.load(out)
    for r in res[1:]:
        assert torch.equal(r, res[0]), "ranks disagree"
    F, zs = _problem(seed)
    R, n = F.shape[0], F.shape[0] // 2
    ranks = res[0][:R].numpy()
    akey = res[0][R:2 * R].numpy().view(np.uint64)
    want = Odom.non_dominated_sort(F, stop_at=n)
    assert np.array_equal(ranks, want)
    # single-process full-range association keys of the candidate rows
    l = Odom.split_fronts(want, n).l
    cand = np.nonzero(want <= l)[0]
    t = (F[cand] @ zs.T).astype(np.float32)
    best = np.argmax(t, axis=1)
    from shard_emulator import f2ord
    keys = (f2ord(t[np.arange(len(cand)), best]) << np.uint64(32)) | (np.uint64(0xFFFFFFFF) -
                                                                     best.astype(np.uint64))
    assert np.array_equal(akey[cand], keys)
    assert (akey[np.setdiff1d(np.arange(R), cand)] == 0).all()
