"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the NSGA-III hot path.

``oracle/manyobj_ref`` is a from-scratch numpy restatement of the behavioural
contract ``/root/reference/SPEC.md`` (the reference ships a specification and
``pkg/src/manyobj/errors.py`` only).  ``oracle/c`` is a C
(OpenMP) restatement of the O(R^2) pieces (dominance, peeling, association)
used to check the numpy oracle at larger sizes and as the multi-core CPU
baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything under ``oracle/``, and only as the
checker or the timed CPU reference — never as part of the product path
(``paper_2504_06067_b200``), which fails loudly when its CUDA library is absent.

Parity pinning: the reference has no tests and no runnable implementation, so
the only golden vectors are SPEC.md's worked examples ([TRIVIAL]/[DERIVED]
tags).  The oracle is pinned against every one of them
(``tests/golden/spec_examples.json``, produced by
``tests/golden/make_golden.py``; checked by ``tests/test_oracle_golden.py``).
Beyond those examples the bit-level arithmetic (FP32 canonical association,
FP64 intercept solve, Philox streams, keyed swap-or-not shuffles) is pinned by this
oracle itself — see DESIGN.md §"Pinned semantics".
"""
