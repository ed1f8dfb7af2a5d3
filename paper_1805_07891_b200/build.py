"""Build libphub.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python paper_1805_07891_b200/build.py          # build if stale (no package import)
    python paper_1805_07891_b200/build.py --force

The .so lands next to this file so it travels with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libphub.so")
LOG = os.path.join(ROOT, "build", "ptxas.log")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(LOG), exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-o", tmp, *sources()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(LOG, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {LOG}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "phub_c_example.c")
EXAMPLE_BIN = os.path.join(ROOT, "build", "phub_c_example")


def build_example() -> str:
    """Compile the plain-C client of the ABI (examples/phub_c_example.c)."""
    os.makedirs(os.path.dirname(EXAMPLE_BIN), exist_ok=True)
    cuda = os.path.dirname(os.path.dirname(nvcc())) if os.path.isabs(nvcc()) else "/usr/local/cuda"
    cmd = ["gcc", "-std=c11", "-Wall", "-O2", "-I", INCLUDE, "-I", os.path.join(cuda, "include"),
           EXAMPLE_SRC, "-L", PKG, "-lphub", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", EXAMPLE_BIN]
    subprocess.check_call(cmd)
    return EXAMPLE_BIN


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
