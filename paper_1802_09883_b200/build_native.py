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
    """Compile the library (to `out`, default LIB) with optional -D defines:
    every .cu to an object in parallel, then one shared-library link."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile

    import time

    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    t_start = time.time()  # the library is stamped with this time: a source edited during the build stays newer
    os.makedirs(os.path.dirname(target), exist_ok=True)
    common = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    tmp = tempfile.mkdtemp(prefix="repro_build_")
    srcs = sources()
    objs = [os.path.join(tmp, os.path.basename(s) + ".o") for s in srcs]

    def compile_one(i):
        return subprocess.run(common + ["-c", srcs[i], "-o", objs[i]], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, range(len(srcs))))
    link = subprocess.run([NVCC, *ARCH, "-shared", *objs, "-o", target + ".tmp"], capture_output=True, text=True)
    log = os.path.join(LIBDIR, "build.log") if out is None else target + ".log"
    with open(log, "w") as fh:
        for s_, r in zip(srcs, results):
            fh.write(" ".join(common + ["-c", s_]) + "\n" + r.stdout + r.stderr)
        fh.write(link.stdout + link.stderr)
    failed = [r for r in results if r.returncode != 0] + ([link] if link.returncode != 0 else [])
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    os.rmdir(tmp)
    if failed:
        sys.stderr.write("".join(r.stdout + r.stderr for r in failed))
        raise RuntimeError("nvcc failed building librepro_b200.so")
    os.replace(target + ".tmp", target)
    os.utime(target, (t_start, t_start))
    if verbose:
        print("".join(r.stderr for r in results))
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
