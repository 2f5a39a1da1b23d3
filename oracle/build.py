"""Build the CPU oracle (oracle/lib/libckks_ref.so) with gcc + OpenMP.
Test infrastructure only."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libckks_ref.so")
SRC = os.path.join(HERE, "ckks_ref.c")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", SRC,
                    "-o", LIB], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
