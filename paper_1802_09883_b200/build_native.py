"""Build the sm_100a shared library in-tree (paper_1802_09883_b200/_lib/).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false, one
.so exporting the C-ABI of include/repro_groupby.h.  Used by
__graft_entry__.build() and by the binding when the library is missing on a
machine with nvcc.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.environ.get("REPRO_B200_LIB") or os.path.join(LIBDIR, "librepro_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "repro_groupby.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library (to `out`, default LIB) with optional -D defines."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-shared", "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, *sources(), "-o", target + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(LIBDIR, "build.log") if out is None else target + ".log"
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building librepro_b200.so")
    os.replace(target + ".tmp", target)
    if verbose:
        print(res.stderr)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
