"""Input coercion shared by the op modules (host plumbing, no arithmetic)."""
import numpy as np
import torch

from .errors import ShapeError


def device():
    return torch.device("cuda", torch.cuda.current_device())


def as_cuda(x, dtype):
    """Contiguous CUDA tensor of ``dtype`` (numpy/lists are copied host->device once)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    if t.dtype != dtype:
        t = t.to(dtype)
    if t.device.type != "cuda":
        t = t.to(device())
    return t.contiguous()


def as_matrix(x, dtype=torch.float32):
    t = as_cuda(x, dtype)
    if t.ndim != 2:
        raise ShapeError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
    return t


def as_mask(valid, n):
    if valid is None:
        return None
    t = as_cuda(valid, torch.uint8)
    if t.shape != (n,):
        raise ShapeError("valid must have one flag per row")
    return t
