"""Can two ranks share one GPU under NCCL here?  torchrun --nproc-per-node 2 scripts/nccl_probe.py"""
import os

import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
x = torch.full((4,), float(r + 1), device="cuda")
out = torch.empty(4 * w, device="cuda")
dist.all_gather_into_tensor(out, x)
y = torch.tensor([r], device="cuda", dtype=torch.int64)
dist.all_reduce(y, op=dist.ReduceOp.MAX)
torch.cuda.synchronize()
print(f"rank {r}: gather {out.tolist()} max {int(y)}", flush=True)
dist.destroy_process_group()
