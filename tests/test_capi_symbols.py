"""CPU-side checks of the boundary: the C-ABI library loads and exports every
function include/repro_groupby.h declares (no compute call without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "repro_groupby.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(repro_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("repro_groupby_sum", "repro_acc_create", "repro_acc_deposit", "repro_acc_merge",
                     "repro_acc_finalize", "repro_acc_export", "repro_acc_import", "repro_acc_destroy",
                     "repro_strerror", "repro_baseline_atomic_sum"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_1802_09883_b200 as R  # loads the .so (no CUDA call)
    lib = ctypes.CDLL(R.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    import paper_1802_09883_b200 as R
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_strerror_and_argument_errors_without_gpu():
    import paper_1802_09883_b200 as R
    lib = R._lib
    assert lib.repro_strerror(0) == b"ok"
    assert lib.repro_strerror(-2).startswith(b"key")
    # argument validation happens before any CUDA call
    assert lib.repro_groupby_sum(None, None, -1, 4, 3, 1, None) == R.EINVAL
    assert lib.repro_groupby_sum(None, None, 0, 0, 3, 1, ctypes.c_void_p(8)) == R.EINVAL
    assert lib.repro_groupby_sum(None, None, 0, 4, 5, 1, ctypes.c_void_p(8)) == R.EINVAL
    assert lib.repro_groupby_sum(None, None, 0, 4, 3, 7, ctypes.c_void_p(8)) == R.EINVAL
    assert lib.repro_groupby_sum(None, None, 10, 4, 3, 1, ctypes.c_void_p(8)) == R.EINVAL
    assert lib.repro_acc_create(None, 4, 3, 1) == R.EINVAL
    assert lib.repro_acc_merge(None, None) == R.EINVAL


def test_no_cpu_fallback_in_product_package():
    # the product package must not reach the oracle
    pkg = os.path.join(ROOT, "paper_1802_09883_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "repro_oracle" not in src and "liboracle" not in src, f
