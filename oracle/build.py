"""Build of the CPU oracle liboracle.so -- TEST INFRASTRUCTURE ONLY (plain gcc, no CUDA).

Kept next to the oracle so the product package never references it.  Called by
__graft_entry__.build() (building the checker is not using it), tests/conftest.py and the
oracle's own ctypes binding when the library is missing.
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIBORACLE = os.path.join(HERE, "liboracle.so")


def build_oracle(force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(HERE, "*.c")))
    deps = srcs + glob.glob(os.path.join(HERE, "*.h")) + [os.path.abspath(__file__)]
    stale = not os.path.exists(LIBORACLE) or any(
        os.path.getmtime(d) > os.path.getmtime(LIBORACLE) for d in deps)
    if force or stale:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", "-o", LIBORACLE, *srcs, "-lm"]
        r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("oracle build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return LIBORACLE


if __name__ == "__main__":
    import sys
    print("built", build_oracle(force="--force" in sys.argv))
