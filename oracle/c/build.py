"""Build oracle/c/liboro.so (gcc -O3 -fopenmp -ffp-contract=off) -- the C/OpenMP restatement used by
tests and bench.py's cpu_baseline only (TEST INFRASTRUCTURE; never loaded by the product)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mo_oracle.c")
SRC3 = os.path.join(HERE, "mo_oracle_nds3.cc")
LIB = os.path.join(HERE, "liboro.so")


def build(force=False):
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(SRC), os.path.getmtime(SRC3))):
        return LIB
    tmp = LIB + ".tmp"
    flags = ["-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC"]
    obj_c, obj_3 = LIB + ".c.o", LIB + ".nds3.o"
    subprocess.run(["gcc", *flags, "-c", SRC, "-o", obj_c], check=True)
    subprocess.run(["g++", *flags, "-std=c++17", "-c", SRC3, "-o", obj_3], check=True)
    subprocess.run(["g++", "-shared", "-fopenmp", obj_c, obj_3, "-o", tmp, "-lm"], check=True)
    for o in (obj_c, obj_3):
        os.unlink(o)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
