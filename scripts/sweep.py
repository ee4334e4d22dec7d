"""Perf exploration: time the reproducible GroupBy and the atomicAdd baseline
over group counts with inputs generated on the GPU (torch RNG; perf only --
parity is covered by tests/ and bench.py).  Prints one line per point."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_09883_b200 as R  # noqa: E402


def make(n, G, dtype, skew=False, uniform_pm1=False):
    if skew:
        u = torch.rand(n, device="cuda", dtype=torch.float64)
        ranks = torch.arange(1, G + 1, device="cuda", dtype=torch.float64) ** -1.1
        cdf = torch.cumsum(ranks, 0)
        cdf /= cdf[-1].clone()
        keys = torch.searchsorted(cdf, u).clamp_(max=G - 1).to(torch.int32)
    else:
        keys = torch.randint(0, G, (n,), device="cuda", dtype=torch.int32)
    if uniform_pm1:
        return keys, (torch.rand(n, device="cuda", dtype=torch.float64) * 2 - 1).to(dtype)
    e = torch.randint(-20, 21, (n,), device="cuda").to(torch.float64)
    v = (torch.rand(n, device="cuda", dtype=torch.float64) + 1.0) * torch.exp2(e)
    v = v * (torch.randint(0, 2, (n,), device="cuda") * 2 - 1)
    return keys, v.to(dtype)


def timeit(fn, steps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 27)
    ap.add_argument("--groups", type=str, default="1,4,16,64,256,1024,4096,16384,65536,262144,1048576,4194304,16777216")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--fold", type=int, default=3)
    ap.add_argument("--skew", action="store_true")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--nobase", action="store_true", help="skip the atomicAdd baseline")
    ap.add_argument("--pm1", action="store_true", help="values U[-1,1) (config 2)")
    a = ap.parse_args()
    dtype = torch.float64 if a.dtype == "f64" else torch.float32
    dt = R.F64 if a.dtype == "f64" else R.F32
    R.set_kernel_variant(a.variant)
    vsz = 8 if a.dtype == "f64" else 4
    for G in [int(x) for x in a.groups.split(",")]:
        keys, vals = make(a.n, G, dtype, a.skew, a.pm1)
        out = torch.empty(G, dtype=dtype, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = R.make_workspace(a.n, G, a.fold, dt)
        t = timeit(lambda: R.groupby_sum_async(keys, vals, G, a.fold, out, ws, st))
        R.timing_enable(True)
        R.groupby_sum_async(keys, vals, G, a.fold, out, ws, st)
        R.timing_enable(False)
        pk = {k: round(v[1], 4) for k, v in R.timing_collect().items()}
        path = R.last_path()
        tbs = [] if a.nobase else [timeit(lambda: R.baseline_atomic_sum(keys, vals, G, variant=0))]
        try:
            tbs.append(timeit(lambda: R.baseline_atomic_sum(keys, vals, G, variant=1)))
        except R.ReproError:
            pass
        tb = min(tbs) if tbs else float("nan")
        gbs = a.n * (4 + vsz) / (t * 1e-3) / 1e9
        print(f"v{a.variant} path{path} G={G:8d} repro {t:.4f} ms ({gbs:7.1f} GB/s, {gbs / 6554.2:.3f} of HBM)  atomic {tb:.4f} ms  "
              f"slowdown {t / tb:.2f}  kernels {pk}", flush=True)
        assert st.item() == 0


if __name__ == "__main__":
    main()
