#!/usr/bin/env python
"""bench.py -- reproducible GroupBy-SUM on B200 (arxiv 1802.09883 hot path).

`python bench.py --gpus N --steps K --warmup W` prints ONE JSON line (rank 0).
A step is one pass of the whole hot path over one batch of synthetic rows
resident in HBM: load + level index + digit cascade + per-group accumulate
(k_onchip_accumulate), fold of the block partials + Eq. 1 read-out (k_fold),
status word (k_status); at N > 1 also the integer NCCL exchange.

Workload at N=1: BASELINE.json configs[1] (2^27 rows, int32 keys U[0,1024),
fp64 values +-(1+mant) 2^e, e in [-20,20], fold K=3), the config the metric
is quoted on.  At N>1 every rank processes its own 2^27-row shard of the same
generator (weak scaling) and the states are combined with integer all-reduces.

Keys reported beside the contract's: roofline (dominant kernel, CUDA events
on its stream), cpu_baseline (the oracle, host cores), e2e (C-ABI with host
buffers: H2D + compute + D2H in the timed region), baseline_atomic (the
non-reproducible atomicAdd GroupBy on the same GPU) and clocks.

`--impl reference` times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "repro GroupBy-SUM rows/s & HBM GB/s vs roofline; slowdown vs plain fp64 atomicAdd"

WORKLOADS = {
    0: "config0: 2^16 rows, keys U[0,16), fp64 +-(1+mant)2^e e in [-20,20], K=3",
    1: "config1: 2^27 rows, keys U[0,1024), fp64 +-(1+mant)2^e e in [-20,20], K=3 (low-cardinality on-chip path)",
    2: "config2: 2^28 rows, keys U[0,G), fp64 U[-1,1), K=3",
    3: "config3: 2^28 rows, keys Zipf(1.1) over 2^20, fp32 normal*2^e e in [-10,10], K=2",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["repro", "reference"], default="repro")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n-groups", type=int, default=None, help="config 2 group count")
    ap.add_argument("--rows", type=int, default=None, help="override rows per GPU (testing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-atomic-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def shape(args):
    from paper_1802_09883_b200 import synth
    c = synth.CONFIGS[args.config]
    n = args.rows or c["n"]
    G = args.n_groups or c["n_groups"] or 1024
    return n, G, c["fold"], c["dtype"]


def gen(args, rank):
    from paper_1802_09883_b200 import synth
    n, G, K, dt = shape(args)
    if args.config == 0:
        keys, vals = synth.generate(0, n=n, r0=rank * n)
    else:
        keys, vals = synth.generate_chunked(args.config, n, G) if rank == 0 else \
            _gen_shard(args.config, n, G, rank)
    return keys, vals


def _gen_shard(config, n, G, rank):
    from paper_1802_09883_b200 import synth
    vt = np.float32 if synth.CONFIGS[config]["dtype"] == "f32" else np.float64
    keys = np.empty(n, np.int32)
    vals = np.empty(n, vt)
    ch = 1 << 24
    for a in range(0, n, ch):
        b = min(n, a + ch)
        if config == 3:
            seed = synth.SEED_BASE + 3
            keys[a:b] = synth.keys_zipf(seed, rank * n + a, rank * n + b, G)
            vals[a:b] = synth.values_normal_exp(seed, rank * n + a, rank * n + b)
        else:
            k, v = synth.generate(config, n=b - a, n_groups=G, r0=rank * n + a)
            keys[a:b], vals[a:b] = k, v
    return keys, vals


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(f"config{config}")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, local_rank):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = local_rank
            if vis and all(x.strip().isdigit() for x in vis.split(",")):
                idx = int(vis.split(",")[local_rank])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def run_oracle(keys, vals, G, K):
    import oracle as O
    threads = O.default_threads()
    t0 = time.perf_counter()
    rc, out = O.groupby_sum(keys, vals, G, K, threads=threads)
    dt = time.perf_counter() - t0
    return rc, out, dt, threads


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands, timed on the host cores
    (rank 0 only; other ranks exit without work).  Each step is a bounded
    sample of the workload -- consecutive row blocks of it -- sized so that all
    K steps together process at most 2^28 rows (a few minutes at worst)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    n, G, K, dt = shape(args)
    steps = max(1, args.steps)
    sample = max(1 << 12, min(n, (1 << 28) // steps))
    rows_needed = min(n, sample * steps)
    args_rows = args.rows
    args.rows = rows_needed
    keys, vals = gen(args, 0)
    args.rows = args_rows
    threads = O.default_threads()
    for w in range(args.warmup):
        O.groupby_sum(keys[: 1 << 12], vals[: 1 << 12], G, K, threads=threads)
    times = []
    for s in range(steps):
        a = (s * sample) % max(1, rows_needed - sample + 1)
        t0 = time.perf_counter()
        rc, _ = O.groupby_sum(keys[a:a + sample], vals[a:a + sample], G, K, threads=threads)
        times.append(time.perf_counter() - t0)
        if rc != 0:
            raise SystemExit(f"oracle status {rc}")
    total = sum(times)
    value = sample * steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": total / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": WORKLOADS.get(args.config), "rows_per_step": sample, "n_groups": G, "fold": K},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "oracle",
                         "sample": f"{sample} consecutive rows of the workload per step"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_1802_09883_b200 as R

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n, G, K, dts = shape(args)
    dt = R.F64 if dts == "f64" else R.F32
    vsz = 8 if dt == R.F64 else 4
    keys_h, vals_h = gen(args, rank)
    keys = torch.from_numpy(keys_h).cuda()
    vals = torch.from_numpy(vals_h).cuda()
    stream = torch.cuda.current_stream()
    out = torch.empty(G, dtype=vals.dtype, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = R.make_workspace(n, G, K, dt)

    from paper_1802_09883_b200 import dist as rdist
    acc = R.Accumulator(G, K, dt) if world > 1 else None

    def step():
        if world == 1:
            R.groupby_sum_async(keys, vals, G, K, out, ws, status, stream)
            return 3
        acc.reset()
        acc.deposit(keys, vals)
        rdist.allreduce_state(acc)
        acc.finalize(out)
        return 0

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    if int(status.item()) != 0:
        raise SystemExit(f"device status {status.item()}")

    # ---- timed region ------------------------------------------------------
    R.timing_enable(True)
    R.timing_collect()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            launches += step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    R.timing_enable(False)
    per_kernel = R.timing_collect()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = sum(c for c, _ in per_kernel.values())  # kernels of librepro_b200 in the timed region
    ms_per_step = ms / args.steps
    rows_total = n * world
    value = rows_total / (ms_per_step * 1e-3)

    # ---- dominant kernel roofline -----------------------------------------
    peak, peak_src = peaks()
    dom = max(per_kernel.items(), key=lambda kv: kv[1][1]) if per_kernel else None
    roof = None
    if dom:
        name, (cnt, kms) = dom
        avg_ms = kms / cnt
        alg_bytes = n * (4 + vsz)  # the kernel's algorithmic input bytes per launch
        achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
        tr = ncu_traffic(args.config)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr, "kernel": name, "kernel_ms": avg_ms,
                "kernel_share_of_step": kms / ms if ms else None, "alg_bytes_per_launch": alg_bytes,
                "peak_source": peak_src}
    step_bytes = n * (4 + vsz) + G * vsz
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dts, "data": "synthetic",
        "config": {"workload": WORKLOADS.get(args.config), "rows_per_gpu": n, "n_groups": G, "fold": K,
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": f"inputs {n * (4 + vsz) / 1e9:.2f} GB/GPU > 126 MB L2 (no flush needed)"},
        "step_hbm_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
        "step_roofline_frac": (step_bytes / (ms_per_step * 1e-3) / 1e9) / peak,
        "roofline": roof,
        "per_kernel_ms": {k: v[1] / v[0] for k, v in per_kernel.items()},
        "gpu_launches": launches,
        "clocks": clk.result(),
    }

    # ---- non-reproducible atomicAdd baseline on the same GPU -------------------
    if not args.no_atomic_baseline and world == 1:
        best = None
        for variant in (0, 1):
            try:
                for _ in range(3):
                    R.baseline_atomic_sum(keys, vals, G, variant=variant, out=None, stream=stream)
                torch.cuda.synchronize()
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                bsteps = max(10, args.steps // 4)
                b0.record(stream)
                for _ in range(bsteps):
                    R.baseline_atomic_sum(keys, vals, G, variant=variant, stream=stream)
                b1.record(stream)
                torch.cuda.synchronize()
                bms = b0.elapsed_time(b1) / bsteps
                if best is None or bms < best[1]:
                    best = (variant, bms)
            except R.ReproError:
                continue
        if best:
            line["baseline_atomic"] = {"variant": ["global_atomicAdd", "smem_privatised_atomicAdd"][best[0]],
                                       "ms_per_step": best[1], "rows_per_s": n / (best[1] * 1e-3),
                                       "slowdown_repro_vs_atomic": ms_per_step / best[1]}

    # ---- end-to-end through the C-ABI with host buffers ---------------------
    if not args.no_e2e and world == 1:
        kp = torch.from_numpy(keys_h).pin_memory()
        vp = torch.from_numpy(vals_h).pin_memory()
        R.groupby_sum_host(kp, vp, G, K)
        e2e_steps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = R.groupby_sum_host(kp, vp, G, K)
        et = (time.perf_counter() - t0) / e2e_steps
        line["e2e"] = {"value": n / et, "unit": "rows/s", "h2d_bytes_per_step": n * (4 + vsz),
                       "d2h_bytes_per_step": G * vsz, "ms_per_step": et * 1e3, "steps": e2e_steps,
                       "bit_identical_to_device_path": bool(torch.equal(res, out.cpu()))}
        del kp, vp

    # ---- oracle: cpu_baseline + parity on this input ---------------------
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rc, ref, t, threads = run_oracle(keys_h, vals_h, G, K)
        got = out.cpu().numpy()
        line["cpu_baseline"] = {"value": n / t, "unit": "rows/s", "cores": threads, "kind": "oracle",
                                "sample": f"the full workload ({n} rows), {threads} host threads",
                                "seconds": t}
        if not args.no_parity:
            line["parity"] = {"vs_oracle": "bit-exact" if (rc == 0 and got.tobytes() == ref.tobytes())
                              else "MISMATCH", "groups": G}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
