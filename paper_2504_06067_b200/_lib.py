"""ctypes binding of libmanyobj_b200.so (the C-ABI in include/manyobj_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, :func:`lib` raises ``RuntimeError`` and every GPU op fails loudly.
"""
import ctypes
import os
import threading

import torch

from .errors import raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmanyobj_b200.so")

_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_u32, c_u64, c_f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_float
c_vp, c_sz = ctypes.c_void_p, ctypes.c_size_t

INFO = dict(L=0, SELECTED=1, K=2, NFRONTS=3, FL_SIZE=4, SKIPPED=5, NEAREST=6, LEVEL=7, SINGULAR=8,
            SURVIVORS=9, ERROR=10, ASSOC_FALLBACK=11, ERROR_FIRST=12)
INFO_COUNT = 16
PHASE_VARY, PHASE_SORT, PHASE_NICHE, PHASE_ALL = 1, 2, 4, 7
NICHE_PREP, NICHE_ASSOC, NICHE_FINISH = 8, 16, 32
SORT_BITS, SORT_STREAM = 0, 1
PROBLEM_IDS = {f"DTLZ{i}": i for i in range(1, 8)}
DROPPED = 2 ** 31 - 1


class VarCfg(ctypes.Structure):
    _fields_ = [("eta_c", c_f32), ("eta_m", c_f32), ("p_c", c_f32), ("p_m", c_f32)]


class StepArgs(ctypes.Structure):
    _fields_ = [
        ("problem", c_i32), ("m", c_i32), ("d", c_i32), ("pad0", c_i32),
        ("n", c_i64), ("w", c_i64), ("seed", c_u64), ("generation", c_u32), ("pad1", c_u32),
        ("var", VarCfg),
        ("zhat", c_vp), ("XR", c_vp), ("FR", c_vp), ("X_next", c_vp), ("F_next", c_vp),
        ("ideal", c_vp), ("ranks", c_vp), ("info", c_vp), ("workspace", c_vp), ("workspace_bytes", c_sz),
        ("generation_dev", c_vp),
        ("sort_mode", c_i32), ("shard_rank", c_i32), ("shard_count", c_i32), ("pad2", c_i32),
        ("lattice_z", c_vp), ("lattice_index", c_vp), ("lattice_pos", c_vp), ("lattice_H", c_i32),
        ("lattice_r", c_i32), ("pad3", c_i32),
        ("zhat_frag", c_vp), ("zhat_umma", c_vp), ("ref_H_outer", c_i32), ("ref_H_inner", c_i32),
    ]


_PROTOS = {
    "mo_version": (ctypes.c_char_p, []),
    "mo_step_args_bytes": (c_sz, []),
    "mo_bits_words_per_row": (c_i64, [c_i64]),
    "mo_trace_offset": (c_i64, [c_i64, c_i32, c_i64]),
    "mo_workspace_bytes": (c_i32, [c_i64, c_i32, c_i32, c_i64, ctypes.POINTER(c_sz)]),
    "mo_workspace_bytes_rows": (c_i32, [c_i64, c_i32, c_i64, ctypes.POINTER(c_sz)]),
    "mo_permutation": (c_i32, [c_i64, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp]),
    "mo_init_population": (c_i32, [c_vp, c_i64, c_i32, c_u64, c_vp]),
    "mo_dtlz_eval": (c_i32, [c_i32, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "mo_vary_eval": (c_i32, [c_i32, c_vp, c_i64, c_i32, c_i32, c_u64, c_u32, ctypes.POINTER(VarCfg),
                             c_vp, c_vp, c_vp, c_vp]),
    "mo_dominance_bits": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "mo_front_peel": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "mo_presort": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "mo_dominance_bits_sorted": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "mo_dominance_tables_bytes": (c_sz, [c_i64, c_i32]),
    "mo_dominance_bits_ranked": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_sz, c_vp,
                                         c_vp]),
    "mo_tile_summary_words": (c_i64, [c_i64]),
    "mo_normalize": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_u64, c_u32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "mo_associate": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_u64, c_u32, c_vp, c_vp, c_vp, c_sz,
                             c_vp]),
    "mo_niche_select": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_u64, c_u32, c_vp, c_vp, c_sz,
                                c_vp]),
    "mo_step": (c_i32, [ctypes.POINTER(StepArgs), c_vp]),
    "mo_select": (c_i32, [ctypes.POINTER(StepArgs), c_vp]),
    "mo_step_phases": (c_i32, [ctypes.POINTER(StepArgs), c_u32, c_vp]),
    "mo_peak_issue": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "mo_niche_phases": (c_i32, [ctypes.POINTER(StepArgs), c_u32, c_vp]),
    "mo_igd_workspace_bytes": (c_sz, [c_i64]),
    "mo_igd": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_vp, c_sz, c_vp]),
    "mo_hv_mc_workspace_bytes": (c_sz, [c_i64]),
    "mo_hv_mc": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_i64, c_u64, c_vp, c_vp, c_sz, c_vp]),
    "mo_hv_exact_workspace_bytes": (c_sz, [c_i64]),
    "mo_pack_refs_bytes": (c_sz, [c_i64]),
    "mo_pack_refs_bf16": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "mo_pack_refs_f16_bytes": (c_sz, [c_i64, c_i32]),
    "mo_pack_refs_f16": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "mo_hv_exact": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "mo_sort_stream_begin": (c_i32, [ctypes.POINTER(StepArgs), c_vp]),
    "mo_sort_stream_front": (c_i32, [ctypes.POINTER(StepArgs), c_i32, c_vp]),
    "mo_sort_stream_end": (c_i32, [ctypes.POINTER(StepArgs), c_vp]),
    "mo_workspace_init": (c_i32, [c_vp, c_sz, c_vp]),
    "mo_stream_stats_offset": (c_i32, [c_i64, c_i32, c_i64, c_i32, c_i32, ctypes.POINTER(c_i64)]),
    "mo_workspace_bytes_ex": (c_i32, [c_i64, c_i32, c_i32, c_i64, c_i32, c_i32, ctypes.POINTER(c_sz)]),
    "mo_stream_offsets": (c_i32, [c_i64, c_i32, c_i64, c_i32, c_i32, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                  ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "mo_niche_offsets": (c_i32, [c_i64, c_i32, c_i64, c_i32, c_i32, ctypes.POINTER(c_i64)]),
    # op-level API (k_ops.cu)
    "mo_ops_workspace_bytes": (c_i32, [c_i64, c_i64, ctypes.POINTER(c_sz)]),
    "mo_step_mask": (c_i32, [c_vp, c_i64, c_vp, c_vp]),
    "mo_masked_argmin": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "mo_segment_count": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "mo_associate_matrix": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "mo_niche_counts": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "mo_nearest_selection": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                                     c_vp, c_vp, c_sz, c_vp]),
    "mo_build_cache": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "mo_batched_random_selection": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz,
                                            c_vp]),
    "mo_sbx_pairs": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, ctypes.c_double, c_f32, ctypes.c_double,
                             ctypes.c_double, c_i32, c_u64, c_u32, c_vp, c_vp, c_vp]),
    "mo_polynomial_mutation": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, ctypes.c_double, c_f32, ctypes.c_double,
                                       ctypes.c_double, c_u64, c_u32, c_vp, c_vp]),
}

EXPORTED = tuple(_PROTOS)


def load_library(path=LIB_PATH):
    """dlopen the library and bind every prototype (no GPU needed)."""
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -m paper_2504_06067_b200.build` "
                           "(the engine has no CPU fallback)")
    so = ctypes.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    return so


def lib():
    """The loaded library; requires a CUDA device (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not torch.cuda.is_available():
                    raise RuntimeError("manyobj_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
                torch.cuda.init()
                _lib = load_library()
    return _lib


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_vp(s.cuda_stream)


def ptr(t):
    return c_vp(0) if t is None else c_vp(t.data_ptr())


def check(code, what):
    raise_for_status(int(code), what)


def workspace_rows(R, m, w, device=None):
    nbytes = c_sz(0)
    check(lib().mo_workspace_bytes_rows(int(R), int(m), int(w), ctypes.byref(nbytes)), "mo_workspace_bytes_rows")
    return torch.empty(int(nbytes.value), dtype=torch.uint8, device=device or "cuda")


def workspace_ops(R, w, device=None):
    nbytes = c_sz(0)
    check(lib().mo_ops_workspace_bytes(int(R), int(w), ctypes.byref(nbytes)), "mo_ops_workspace_bytes")
    return torch.empty(max(1, int(nbytes.value)), dtype=torch.uint8, device=device or "cuda")


def workspace_step(n, m, d, w, device=None):
    nbytes = c_sz(0)
    check(lib().mo_workspace_bytes(int(n), int(m), int(d), int(w), ctypes.byref(nbytes)), "mo_workspace_bytes")
    return torch.zeros(int(nbytes.value), dtype=torch.uint8, device=device or "cuda")   # mo_workspace_init


def workspace_bytes_ex(n, m, d, w, sort_mode, shards):
    nbytes = c_sz(0)
    check(load_library_cached().mo_workspace_bytes_ex(int(n), int(m), int(d), int(w), int(sort_mode), int(shards),
                                                      ctypes.byref(nbytes)), "mo_workspace_bytes_ex")
    return int(nbytes.value)


def stream_offsets(n, m, w, sort_mode, shards):
    """(mask_local byte offset, mask_local words, mask_full byte offset, akey byte offset) in the workspace."""
    out = [c_i64(0) for _ in range(4)]
    check(load_library_cached().mo_stream_offsets(int(n), int(m), int(w), int(sort_mode), int(shards),
                                                  *[ctypes.byref(o) for o in out]), "mo_stream_offsets")
    return tuple(int(o.value) for o in out)


def niche_offsets(n, m, w, sort_mode, shards):
    """Byte offsets of the niche state of one step in the workspace (mo_niche_offsets)."""
    out = (c_i64 * 11)()
    check(load_library_cached().mo_niche_offsets(int(n), int(m), int(w), int(sort_mode), int(shards), out),
          "mo_niche_offsets")
    keys = ("pi", "d", "rho", "rho_p", "take", "kept", "prom", "pos_pop", "perm_pop", "pos_ref", "perm_ref")
    return dict(zip(keys, (int(x) for x in out)))


_host_lib = None


def load_library_cached():
    """The library for sizing queries only (no device needed); compute calls go through lib()."""
    global _host_lib
    if _lib is not None:
        return _lib
    if _host_lib is None:
        _host_lib = load_library()
    return _host_lib


def new_info(device=None, **fields):
    info = torch.zeros(INFO_COUNT, dtype=torch.int32)
    for k, v in fields.items():
        info[INFO[k]] = int(v)
    return info.to(device or "cuda")
