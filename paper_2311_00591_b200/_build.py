"""In-tree build of the native libraries (no JIT cache: the .so files travel with the repo).

  paper_2311_00591_b200/libcoop.so  -- the product: CUDA kernels + C ABI (include/coop.h)
  gen/libcoopgen.so                 -- seeded input generators (host + device)

The CPU oracle (test infrastructure) has its own build next to it (oracle/build.py).
"""
from __future__ import annotations

import glob
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2311_00591_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# bit-exact fp64 paths: no FMA contraction on device or host (R1)
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-shared",
                     "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-O3"]

LIBCOOP = os.path.join(PKG, "libcoop.so")
LIBGEN = os.path.join(ROOT, "gen", "libcoopgen.so")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def build_libcoop(force: bool = False) -> str:
    cu = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    deps = cu + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(
        os.path.join(PKG, "csrc", "*.h")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    if force or _stale(LIBCOOP, deps):
        _run([NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I",
              os.path.join(PKG, "csrc"), "-o", LIBCOOP, *cu])
    return LIBCOOP


def build_libgen(force: bool = False) -> str:
    src = [os.path.join(ROOT, "gen", "coop_gen.cu"), os.path.join(ROOT, "gen", "coop_gen.h")]
    if force or _stale(LIBGEN, src):
        _run([NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "gen"), "-o", LIBGEN, src[0]])
    return LIBGEN


def build_all(force: bool = False) -> None:
    build_libcoop(force)
    build_libgen(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print("built", LIBCOOP, LIBGEN)
