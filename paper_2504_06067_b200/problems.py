"""DTLZ1-7 evaluation on the GPU (DTLZ1/4/6 per the standard suite)."""
from dataclasses import dataclass

import torch

from . import _lib
from ._tensor import as_matrix
from .errors import DomainError, ParameterError, ShapeError

KINDS = tuple(_lib.PROBLEM_IDS)


@dataclass(frozen=True)
class ContinuousProblem:
    """kind, m objectives, d >= m variables in [0,1]^d."""
    kind: str
    m: int
    d: int

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ParameterError(f"unknown problem {self.kind}")
        if self.m < 2 or self.d < self.m:
            raise ParameterError("need m >= 2 and d >= m")

    @property
    def id(self):
        return _lib.PROBLEM_IDS[self.kind]


def dtlz_eval(problem, X):
    """Objective matrix (n x m FP32 CUDA tensor) of ``problem`` at X.

    Raises DomainError when any x lies outside [0,1] (checked on the device,
    read back once).
    """
    X = as_matrix(X)
    n, d = X.shape
    if d != problem.d:
        raise ShapeError("X must be n x d")
    F = torch.empty((n, problem.m), dtype=torch.float32, device=X.device)
    flag = torch.zeros(1, dtype=torch.int32, device=X.device)
    _lib.check(_lib.lib().mo_dtlz_eval(problem.id, _lib.ptr(X), n, d, problem.m, _lib.ptr(F), _lib.ptr(flag),
                                       _lib.stream_ptr()), "mo_dtlz_eval")
    if int(flag.item()):
        raise DomainError("x outside [0,1]^d")
    return F
