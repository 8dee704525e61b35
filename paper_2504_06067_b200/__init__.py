"""paper_2504_06067_b200 -- B200-native NSGA-III survivor selection + variation.

Drop-in for the ``manyobj`` package of arxiv 2504.06067 (TensorNSGA-III) on its
hot path: ``engine.initialize/step/run`` plus the dominance / niche /
variation / problems ops, all backed by hand-written sm_100a kernels in
``libmanyobj_b200.so`` (C-ABI: include/manyobj_b200.h).  ``import
paper_2504_06067_b200 as manyobj`` gives the reference module layout.
"""
from . import errors  # noqa: F401  (no CUDA needed)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy submodule import: the GPU modules pull in torch
    import importlib
    if name in ("batchcore", "bench", "cli", "dominance", "engine", "metrics", "niche", "problems", "refpoints",
                "variation"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
