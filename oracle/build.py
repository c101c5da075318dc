"""Build the oracle's C restatements (TEST INFRASTRUCTURE ONLY) with gcc.

    python oracle/build.py

Output: ``oracle/liboracle.so`` (git-ignored; travels to the GPU box with the
snapshot like the backend's own library).  Called by ``__graft_entry__.build()``.
The reference is pure Python, so there is no ``oracle/_ref`` build.
"""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SOURCES = [os.path.join(HERE, "csrc", "spmv_csr.c")]


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and all(os.path.getmtime(s) <= os.path.getmtime(LIB) for s in SOURCES):
        return LIB
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", *SOURCES, "-o", LIB]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
