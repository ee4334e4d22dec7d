"""Phase profile of the routed kernel (k_route.cu) from an RT_PROF=1 build:
python scripts/rt_prof.py [G ...] (config-2 values, 2^28 rows; Zipf config-3
shape with 'z')."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09883_b200 as R  # noqa: E402

lib = R._lib
prof = getattr(lib, "repro_debug_route_prof", None)
n = int(os.environ.get("RT_N", str(1 << 28)))
args = sys.argv[1:] or ["16384", "65536", "z"]
for a in args:
    torch.manual_seed(0)
    if a == "z":
        G = 1 << 20
        p = torch.arange(1, G + 1, dtype=torch.float64, device="cuda") ** -1.1
        cdf = torch.cumsum(p / p.sum(), 0)
        keys = torch.searchsorted(cdf, torch.rand(n, dtype=torch.float64, device="cuda")).clamp_(max=G - 1).int()
        vals = (torch.randn(n, device="cuda") * torch.exp2(torch.randint(-10, 11, (n,), device="cuda").float()))
        K = 2
    else:
        G = int(a)
        keys = torch.randint(0, G, (n,), dtype=torch.int32, device="cuda")
        vals = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
        K = 3
    out = R.groupby_sum(keys, vals, G, K)
    torch.cuda.synchronize()
    if prof:
        buf = (ctypes.c_ulonglong * 16)()
        prof(buf)
    R.timing_enable(True)
    for _ in range(3):
        R.groupby_sum(keys, vals, G, K, out=out)
    torch.cuda.synchronize()
    t = R.timing_collect()
    R.timing_enable(False)
    line = {k: round(v[1] / v[0], 3) for k, v in t.items()}
    if prof:
        prof(buf)
        nb = max(1, buf[0])
        cyc = {name: buf[i] / nb / 1.965e6 for i, name in
               [(1, "p_rank"), (4, "p_resv"), (5, "p_stage"), (6, "p_write"), (2, "c_wait"), (3, "c_dep")]}
        line["ms_per_block"] = {k: round(v, 3) for k, v in cyc.items()}
        line["per_block"] = {"slow_tiles": buf[8] / nb, "defer_loops": buf[9] / nb, "write_passes": buf[10] / nb,
                             "probe_waits_w0": buf[11] / nb}
    print(a, line, flush=True)
