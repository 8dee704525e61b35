"""The C-ABI library loads and exports every symbol include/manyobj_b200.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2504_06067_b200 import _lib, errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "manyobj_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(mo_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2504_06067_b200 import build
        build.build()
    return _lib.load_library()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("mo_step", "mo_select", "mo_dominance_bits", "mo_front_peel", "mo_associate", "mo_niche_select",
              "mo_normalize", "mo_vary_eval", "mo_dtlz_eval", "mo_permutation", "mo_workspace_bytes"):
        assert s in syms


def test_library_exports_every_declared_symbol(so):
    for s in declared_symbols():
        assert hasattr(so, s), s
    assert set(_lib.EXPORTED) >= set(declared_symbols())


def test_pure_host_entry_points(so):
    assert b"sm_100a" in so.mo_version()
    assert so.mo_bits_words_per_row(1) == 8
    assert so.mo_bits_words_per_row(257) == 16
    nbytes = ctypes.c_size_t(0)
    assert so.mo_workspace_bytes(10000, 5, 14, 8855, ctypes.byref(nbytes)) == 0
    W = so.mo_bits_words_per_row(20000)
    assert nbytes.value >= 20000 * W * 4
    assert so.mo_workspace_bytes(0, 5, 14, 8855, ctypes.byref(nbytes)) == 2


def test_status_codes_map_to_reference_errors():
    assert errors.STATUS_TO_ERROR[1] is errors.ShapeError
    assert errors.STATUS_TO_ERROR[6] is errors.InfeasibleSplitError
    with pytest.raises(errors.ParameterError):
        errors.raise_for_status(2, "x")
    errors.raise_for_status(0, "ok")


def test_step_args_layout_matches_header(so):
    # offsets of the ctypes mirror must match the C struct (natural alignment, 8-byte pointers)
    A = _lib.StepArgs
    assert A.n.offset == 16 and A.seed.offset == 32 and A.var.offset == 48 and A.zhat.offset == 64
    assert A.generation_dev.offset == A.workspace_bytes.offset + 8
    assert A.pad3.offset == A.lattice_r.offset + 4 and A.zhat_frag.offset % 8 == 0
    assert A.zhat_umma.offset == A.zhat_frag.offset + 8
    assert A.ref_H_outer.offset == A.zhat_umma.offset + 8 and A.ref_H_inner.offset == A.ref_H_outer.offset + 4
    assert ctypes.sizeof(A) == A.ref_H_inner.offset + 4
    so.mo_step_args_bytes.restype = ctypes.c_size_t
    assert so.mo_step_args_bytes() == ctypes.sizeof(A)
