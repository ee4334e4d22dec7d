"""Debug builds (-DTAB_DEBUG=1): calls per k_table mode (slow, band, uniform)
for a few GroupBy shapes."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09883_b200 as R  # noqa: E402

lib = ctypes.CDLL(R.LIB_PATH)
out = (ctypes.c_ulonglong * 3)()
for n, G, pm1 in [(1 << 27, 1024, False), (1 << 28, 4096, True), (1 << 28, 1024, True), (1 << 26, 2048, True)]:
    keys = torch.randint(0, G, (n,), device="cuda", dtype=torch.int32)
    if pm1:
        vals = torch.rand(n, device="cuda", dtype=torch.float64) * 2 - 1
    else:
        e = torch.randint(-20, 21, (n,), device="cuda").to(torch.float64)
        vals = (torch.rand(n, device="cuda", dtype=torch.float64) + 1) * torch.exp2(e)
    lib.repro_debug_table_modes(out)
    R.groupby_sum(keys, vals, G, 3)
    lib.repro_debug_table_modes(out)
    print(f"n={n} G={G} pm1={pm1}: slow {out[0]} band {out[1]} uniform {out[2]}", flush=True)
