"""Build libmanyobj_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

``python -m paper_2504_06067_b200.build [--verbose]``.  The .so lands next to
this file so it travels to the GPU box with the gpurun snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmanyobj_b200.so")
SOURCES = ["mo_capi.cu", "k_vary.cu", "k_dominance.cu", "k_stream.cu", "k_niche.cu", "k_metrics.cu", "k_peaks.cu", "k_ops.cu", "k_dom_rank.cu", "k_assoc_umma.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",               # pinned arithmetic: no mul+add contraction anywhere
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "manyobj_b200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(verbose=False, force=False):
    """Compile every source to an object in parallel (one nvcc per file), then link the .so."""
    from concurrent.futures import ThreadPoolExecutor
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f not in ("-shared",)]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *cflags, "-c"] + (["-Xptxas", "-v"] if verbose else []) + \
              ["-o", obj, os.path.join(CSRC, src)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for obj, res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {obj}:\n" + res.stdout + res.stderr)
        if verbose:
            sys.stderr.write(res.stderr)
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp"] + [o for o, _ in results]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
