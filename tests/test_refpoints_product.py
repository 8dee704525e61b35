"""The product's reference-point module (paper_2504_06067_b200/refpoints.py, host setup run once per
Engine) against SPEC.md:112-138's worked examples and, point for point, against the oracle's
independent restatement (oracle/manyobj_ref/refpoints.py) -- the Z the GPU engine uploads is the
Z the oracle checks with.  CPU only."""
import numpy as np
import pytest

from conftest import examples
from oracle.manyobj_ref import refpoints as Oref
from paper_2504_06067_b200 import errors
from paper_2504_06067_b200 import refpoints as P


@pytest.mark.parametrize("ex", examples({"das_dennis", "das_dennis_count", "two_layer_count", "two_layer_contains",
                                         "choose_divisions", "choose_divisions_le"}), ids=lambda e: e["line"])
def test_product_refpoints_spec_examples(ex):
    op = ex["op"]
    if op == "das_dennis":
        if "error" in ex:
            with pytest.raises(getattr(errors, ex["error"])):
                P.das_dennis(ex["m"], ex["H"])
            return
        got = P.das_dennis(ex["m"], ex["H"])
        assert sorted(map(tuple, got.tolist())) == sorted(map(tuple, ex["out"]))
    elif op == "das_dennis_count":
        assert len(P.das_dennis(ex["m"], ex["H"])) == ex["count"]
    elif op == "two_layer_count":
        Z = P.two_layer(ex["m"], ex["Ho"], ex["Hi"])
        assert len(Z) == ex["count"] == P.lattice_size(ex["m"], ex["Ho"], ex["Hi"])
        assert np.allclose(Z.sum(axis=1), 1.0, atol=1e-12)
    elif op == "two_layer_contains":
        Z = P.two_layer(ex["m"], ex["Ho"], ex["Hi"])
        assert np.isclose(Z, np.array(ex["point"])[None, :], atol=1e-12).all(axis=1).any()
    elif op == "choose_divisions":
        assert list(P.choose_divisions(ex["m"], ex["n"])) == ex["H"]
        assert len(P.reference_points(ex["m"], ex["n"])) == ex["w"]
    elif op == "choose_divisions_le":
        Ho, Hi = P.choose_divisions(ex["m"], ex["n"])
        assert len(P.two_layer(ex["m"], Ho, Hi)) <= ex["w_max"]


CASES = [(m, n) for m in (2, 3, 4, 5) for n in (5, 30, 92, 500, 2000)] + \
        [(6, 132), (8, 300), (8, 1000), (10, 200), (10, 2000), (12, 500), (16, 700)]


@pytest.mark.parametrize("m,n", CASES)
def test_product_refpoints_equal_oracle(m, n):
    assert tuple(P.choose_divisions(m, n)) == tuple(Oref.choose_divisions(m, n))
    Zp, Zo = P.reference_points(m, n), Oref.reference_points(m, n)
    assert Zp.shape == Zo.shape
    assert np.array_equal(Zp, Zo)                                     # same points, same order
    assert np.array_equal(P.unit_directions(Zp), Oref.unit_directions(Zo))


@pytest.mark.parametrize("m,n,w", [(3, 92, 91), (5, 10000, 8855), (10, 100000, 97383), (3, 1000000, 998991)])
def test_baseline_config_reference_sets(m, n, w):
    """the w of C1-C4 (C3 two-layer (10, 6), C4 H = 1412)."""
    assert P.lattice_size(m, *P.choose_divisions(m, n)) == w
    if w < 200000:
        assert np.array_equal(P.reference_points(m, n), Oref.reference_points(m, n))


def test_product_refpoints_errors_match_oracle():
    for m, n in [(5, 4), (1, 10), (0, 3)]:
        with pytest.raises(errors.ParameterError):
            P.choose_divisions(m, n)
        with pytest.raises(errors.ParameterError):
            Oref.choose_divisions(m, n)
