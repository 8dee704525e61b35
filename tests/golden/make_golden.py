"""Write tests/golden/spec_examples.json: every worked example of SPEC.md for the hot path.

The reference (/root/reference) ships a specification plus
pkg/src/manyobj/errors.py and nothing else: these literal examples are its
only golden vectors.  Each record cites the SPEC.md line it transcribes.
Exception names are taken from the reference's own errors module (imported
from /root/reference when present) so the fixture pins the error taxonomy.

Run: python tests/golden/make_golden.py  (needs /root/reference only to
cross-check the exception names; the JSON is committed).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

ERROR_NAMES = ["ShapeError", "ParameterError", "BoundsError", "EmptySelectionError", "DomainError",
               "ConfigError", "InfeasibleSplitError", "ParseError"]


def reference_error_names():
    if not os.path.isdir(REF_SRC):
        return ERROR_NAMES
    sys.path.insert(0, REF_SRC)
    try:
        import manyobj.errors as E  # the reference's only implemented module
        names = [n for n in ERROR_NAMES if isinstance(getattr(E, n, None), type)]
        assert names == ERROR_NAMES, names
        return names
    finally:
        sys.path.remove(REF_SRC)


EXAMPLES = [
    # batchcore
    dict(op="step_mask", line="SPEC.md:46", x=[-1, 0, 2], out=[0, 0, 1]),
    dict(op="step_mask", line="SPEC.md:47", x=[0, 0, 0], out=[0, 0, 0]),
    dict(op="step_mask", line="SPEC.md:48", x=[1, 2.5, 3], out=[1, 1, 1]),
    dict(op="masked_argmin", line="SPEC.md:55", values=[3, 1, 2], valid=[1, 1, 1], out=1),
    dict(op="masked_argmin", line="SPEC.md:56", values=[3, 1, 2], valid=[1, 0, 1], out=2),
    dict(op="masked_argmin", line="SPEC.md:57", values=[3, 1, 2], valid=[0, 0, 0], error="EmptySelectionError"),
    dict(op="segment_count", line="SPEC.md:64", labels=[0, 1, 1, 2], valid=[1, 1, 1, 1], segments=4,
         out=[1, 2, 1, 0]),
    dict(op="segment_count", line="SPEC.md:65", labels=[0, 1, 1, 2], valid=[1, 0, 1, 1], segments=3,
         out=[1, 1, 1]),
    dict(op="segment_count", line="SPEC.md:66", labels=[0, 1, 1, 2], valid=[0, 0, 0, 0], segments=3,
         out=[0, 0, 0]),
    dict(op="shuffle_rows_single", line="SPEC.md:73", rows=1, perm=[0]),
    # refpoints
    dict(op="das_dennis", line="SPEC.md:118", m=2, H=4,
         out=[[0, 1], [0.25, 0.75], [0.5, 0.5], [0.75, 0.25], [1, 0]]),
    dict(op="das_dennis", line="SPEC.md:119", m=3, H=1, out=[[0, 0, 1], [0, 1, 0], [1, 0, 0]]),
    dict(op="das_dennis_count", line="SPEC.md:120", m=3, H=12, count=91),
    dict(op="das_dennis", line="SPEC.md:116", m=1, H=3, error="ParameterError"),
    dict(op="two_layer_count", line="SPEC.md:127", m=3, Ho=1, Hi=0, count=3),
    dict(op="two_layer_count", line="SPEC.md:128", m=3, Ho=2, Hi=1, count=9),
    dict(op="two_layer_contains", line="SPEC.md:129", m=3, Ho=1, Hi=1, point=[2 / 3, 1 / 6, 1 / 6]),
    dict(op="choose_divisions", line="SPEC.md:136", m=3, n=91, H=[12, 0], w=91),
    dict(op="choose_divisions", line="SPEC.md:137", m=2, n=100, H=[99, 0], w=100),
    dict(op="choose_divisions_le", line="SPEC.md:138", m=6, n=132, w_max=132),
    # dominance
    dict(op="dominates", line="SPEC.md:184", a=[1, 2], b=[2, 3], out=True),
    dict(op="dominates", line="SPEC.md:185", a=[1, 3], b=[2, 2], out=False),
    dict(op="dominates", line="SPEC.md:186", a=[2, 2], b=[2, 2], out=False),
    dict(op="dominates", line="SPEC.md:182", a=[1, 2], b=[1, 2, 3], error="ShapeError"),
    dict(op="dominance_matrix", line="SPEC.md:193", F=[[1, 2]], out=[[False]]),
    dict(op="dominance_matrix", line="SPEC.md:194", F=[[0, 0], [1, 1]], out=[[False, True], [False, False]]),
    dict(op="non_dominated_sort", line="SPEC.md:202", F=[[1, 2], [1, 2], [1, 2]], out=[0, 0, 0]),
    dict(op="non_dominated_sort", line="SPEC.md:203", F=[[0, 2], [2, 0], [1, 1], [2, 2]], out=[0, 0, 0, 1]),
    dict(op="non_dominated_sort", line="SPEC.md:204", F=[[0, 0], [1, 1], [2, 2]], out=[0, 1, 2]),
    dict(op="split_fronts", line="SPEC.md:211", sizes=[3, 3, 2], n=4, out=[1, 3, 1]),
    dict(op="split_fronts", line="SPEC.md:212", sizes=[4], n=4, out=[0, 0, 4]),
    dict(op="split_fronts", line="SPEC.md:213", sizes=[5, 5], n=5, out=[0, 0, 5]),
    dict(op="split_fronts", line="SPEC.md:209", sizes=[2], n=4, error="InfeasibleSplitError"),
    # variation
    dict(op="sbx_pair", line="SPEC.md:264", p1=[0.2, 0.7], p2=[0.6, 0.1], u=[0.5, 0.5], eta=20,
         c1=[0.2, 0.7], c2=[0.6, 0.1]),
    dict(op="sbx_sum", line="SPEC.md:265", p1=[0.2, 0.7, 0.4], p2=[0.6, 0.1, 0.4], u=[0.1, 0.9, 0.3], eta=20),
    dict(op="sbx_pair", line="SPEC.md:266", p1=[0.3, 0.3], p2=[0.3, 0.3], u=[0.05, 0.95], eta=20,
         c1=[0.3, 0.3], c2=[0.3, 0.3]),
    dict(op="pm", line="SPEC.md:273", x=[0.2, 0.9], u=[0.5, 0.5], eta=20, out=[0.2, 0.9]),
    dict(op="pm_lower", line="SPEC.md:275", x=[0.0], u=[0.25], eta=20),
    # niche
    dict(op="normalize", line="SPEC.md:337", F=[[1, 0, 0], [0, 1, 0], [0, 0, 1]], ideal=[0, 0, 0],
         out=[[1, 0, 0], [0, 1, 0], [0, 0, 1]], intercepts=[1, 1, 1]),
    dict(op="normalize", line="SPEC.md:338", F=[[3, 5], [3, 5], [3, 5]], ideal=None,
         out=[[0, 0], [0, 0], [0, 0]]),
    dict(op="normalize", line="SPEC.md:339", F=[[2, 4], [4, 2]], ideal=None, out=[[0, 1], [1, 0]],
         ideal_out=[2, 2], intercepts=[2, 2]),
    dict(op="distance", line="SPEC.md:346", f=[1, 1], z=[1, 0], out=1.0),
    dict(op="distance", line="SPEC.md:347", f=[2, 2], z=[1, 1], out=0.0),
    dict(op="distance", line="SPEC.md:348", f=[0, 0], z=[1, 0], out=0.0),
    dict(op="associate", line="SPEC.md:355", D=[[0.3, 0.1, 0.5]], valid=[1], pi=[1], d=[0.1]),
    dict(op="associate", line="SPEC.md:356", D=[[0.2, 0.2, 0.2]], valid=[1], pi=[0], d=[0.2]),
    dict(op="associate", line="SPEC.md:357", D=[[0.2, 0.1], [0.4, 0.3]], valid=[1, 0], pi=[1, -1]),
    dict(op="niche_counts", line="SPEC.md:364", pi=[0, 0, 1, 2], ranks=[0, 1, 1, 1], l=1, w=3,
         rho=[1, 0, 0], rho_p=[1, 1, 1]),
    dict(op="niche_counts", line="SPEC.md:365", pi=[0, 0, 1], ranks=[0, 1, 1], l=1, w=3,
         rho=[1, 0, "inf"], rho_p=[1, 1, 0]),
    dict(op="niche_counts", line="SPEC.md:366", pi=[0, 1], ranks=[0, 0], l=0, w=2, rho=[0, 0], rho_p=[1, 1]),
    dict(op="nearest", line="SPEC.md:373", pi=[0, 0], d=[0.4, 0.2], ranks=[0, 0], l=0, w=1, k=1, out=[1]),
    dict(op="nearest", line="SPEC.md:375", pi=[0, 1], d=[0.4, 0.2], ranks=[0, 0], l=0, w=2, k=2, out=[0, 1]),
    dict(op="build_cache", line="SPEC.md:382", pi=[1, 1, 1, 1, 1, 0, 1, 1, 1, 0], ranks=[0] * 10, l=0, w=2,
         row=0, out=[5, 9]),
    dict(op="batched", line="SPEC.md:391", k=0),
    dict(op="batched_one_point", line="SPEC.md:392", candidates=3, k=2),
    dict(op="oracle_single", line="SPEC.md:400", k=1),
    # engine
    dict(op="engine_config_error", line="SPEC.md:442", field="n", n=91, m=3),
    dict(op="engine_config_error", line="SPEC.md:442", field="generations", n=92, m=3, generations=0),
    # problems
    dict(op="dtlz2_sphere", line="SPEC.md:526", m=3, d=12),
    dict(op="dtlz_point", line="SPEC.md:527", kind="DTLZ2", m=3, d=12, x=[0, 0] + [0.5] * 10, out=[1, 0, 0]),
    dict(op="dtlz7_base", line="SPEC.md:528", m=3, d=22),
    dict(op="dtlz_domain", line="SPEC.md:524", kind="DTLZ2", m=3, d=5, x=[1.5, 0, 0.5, 0.5, 0.5],
         error="DomainError"),
]


def main():
    names = reference_error_names()
    for e in EXAMPLES:
        if "error" in e:
            assert e["error"] in names, e
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump({"source": "/root/reference/SPEC.md worked examples", "errors": names, "examples": EXAMPLES},
                  f, indent=1)


if __name__ == "__main__":
    main()
