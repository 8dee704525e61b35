"""``manyobj_ref`` -- numpy restatement of SPEC.md (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""
from . import batchcore, dominance, engine, niche, problems, refpoints, rng, variation  # noqa: F401
