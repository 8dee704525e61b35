"""Build oracle/c/liboro.so (gcc -O3 -fopenmp -ffp-contract=off) -- the C/OpenMP restatement used by
tests and bench.py's cpu_baseline only (TEST INFRASTRUCTURE; never loaded by the product)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mo_oracle.c")
LIB = os.path.join(HERE, "liboro.so")


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + ".tmp"
    subprocess.run(["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", SRC,
                    "-o", tmp, "-lm"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
