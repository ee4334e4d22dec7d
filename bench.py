#!/usr/bin/env python
"""bench.py -- reproducible GroupBy-SUM on B200 (arxiv 1802.09883 hot path).

`python bench.py --gpus N --steps K --warmup W` prints ONE JSON line (rank 0).
A step is one pass of the whole hot path over one batch of synthetic rows
resident in HBM: load + level index + digit cascade + per-group accumulate
(k_onchip_accumulate, or the partition kernels for high group counts), fold
of the block partials + Eq. 1 read-out (k_fold), status word (k_status); at
N > 1 also the integer NCCL exchange.

Workload at N=1 (default): BASELINE.json configs[1] (2^27 rows, int32 keys
U[0,1024), fp64 values +-(1+mant) 2^e, e in [-20,20], fold K=3), the config
the metric is quoted on.  At N>1 every rank processes its own shard of the
same generator (weak scaling: each rank its own 2^27 rows) and the states are
combined with integer all-reduces (config 4: of the fused pass's slot tables).  `--config 2 --n-groups G`, `--config 3`
and `--config 4` time the other BASELINE configs (parity/sweep runs; config 4
is the multi-column call: 4 reproducible SUMs + COUNT over a row projection).

Keys reported beside the contract's: roofline (dominant kernel, CUDA events
on its stream), cpu_baseline (the oracle, host cores, bounded sample), e2e
(C-ABI with host buffers: H2D + compute + D2H in the timed region),
baseline_atomic (the non-reproducible atomicAdd GroupBy on the same GPU),
parity (bit comparison with the oracle) and clocks.

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
    4: "config4: 2^30 rows, keys U[0,4), fp64 qty/price/disc/tax, 4 repro SUMs (qty, price, price*(1-disc), "
       "price*(1-disc)*(1+tax)) + COUNT, K=3 (fused multi-column pass)",
    5: "f4 sum: 2^28 fp64 values +-(1+mant)2^e e in [-20,20] (config-1 values), keyless reproducible SUM, K=3",
    6: "f4 dot: 2^27 x 2 fp64 vectors +-(1+mant)2^e e in [-20,20], reproducible dot product, K=3",
}
# f1: arbitrary int64 keys -- an extra workload, not a BASELINE config
SPARSE = dict(n=1 << 26, distinct=1 << 18)
WORKLOADS[7] = ("f1 sparse keys: 2^26 rows, int64 keys = SplitMix64 of ids uniform over 2^18 (2^18 distinct "
                "keys spread over int64), fp64 +-(1+mant)2^e e in [-20,20], K=3 (hash-mapped dense path)")
# f4: keyless single-array SUM / dot -- extra workloads, not BASELINE configs
ARRAY = {5: dict(n=1 << 28, dot=False), 6: dict(n=1 << 27, dot=True)}
ORACLE_SAMPLE_ROWS = 1 << 27  # bounded oracle sample (cpu_baseline): <= 2^27 rows, well under 30 s of host work
PARITY_ROWS_MULTI = 1 << 24   # config 4: rows of the full input re-run on both sides for the parity check


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
    ap.add_argument("--no-configs", action="store_true", help="headline workload only (skip the sub-results)")
    return ap.parse_args()


def shape(args):
    from inputs import synth
    if args.config in ARRAY:
        return args.rows or ARRAY[args.config]["n"], 1, 3, "f64"
    c = synth.CONFIGS[args.config]
    n = args.rows or c["n"]
    G = args.n_groups or c["n_groups"] or 1024
    return n, G, c["fold"], c["dtype"]


def host_rows(config, r0, n, G):
    """Host copy of rows [r0, r0+n) of a config (numpy generator)."""
    from inputs import synth
    if config in ARRAY:  # values of config 1 (x) and of a second seed (y); no keys
        cols = [synth.generate(1, n=n, r0=r0)[1]]
        if ARRAY[config]["dot"]:
            cols.append(synth.generate(1, n=n, r0=r0, seed=synth.SEED_BASE + config)[1])
        return None, cols
    if config == 3:
        seed = synth.SEED_BASE + 3
        keys = np.empty(n, np.int32)
        vals = np.empty(n, np.float32)
        cdf = synth.zipf_cdf(G, 1.1)
        ch = 1 << 24
        for a in range(0, n, ch):
            b = min(n, a + ch)
            keys[a:b] = synth.keys_zipf(seed, r0 + a, r0 + b, G, cdf=cdf)
            vals[a:b] = synth.values_normal_exp(seed, r0 + a, r0 + b)
        return keys, [vals]
    if config == 4:
        keys, cols = synth.generate(4, n=n, n_groups=G, r0=r0)
        return keys, list(cols)
    keys = np.empty(n, np.int32)
    vals = np.empty(n, np.float64)
    ch = 1 << 24
    for a in range(0, n, ch):
        b = min(n, a + ch)
        keys[a:b], vals[a:b] = synth.generate(config, n=b - a, n_groups=G, r0=r0 + a)
    return keys, [vals]


def device_rows(R, torch, config, r0, n, G):
    """Device-resident rows: generated on the GPU where the device generator
    exists (configs 0/1/2/4, bit-identical to synth.py), else uploaded."""
    if config in ARRAY:
        from inputs import synth
        cols = [R.synth_generate(1, n, 1024, r0=r0)[1][0]]
        if ARRAY[config]["dot"]:
            cols.append(R.synth_generate(1, n, 1024, r0=r0, seed=synth.SEED_BASE + config)[1][0])
        return None, cols
    if config in (0, 1, 2, 4):
        return R.synth_generate(config, n, G, r0=r0)
    keys, cols = host_rows(config, r0, n, G)
    return torch.from_numpy(keys).cuda(), [torch.from_numpy(c).cuda() for c in cols]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


_FP_RATE = {}


def fp_add_rate(R, dt):
    """Measured adds/s of the value type's FP pipe (repro_measure_fp_add_rate), once per dtype."""
    if dt not in _FP_RATE:
        _FP_RATE[dt] = R.measure_fp_add_rate(dt)
    return _FP_RATE[dt]


def ncu_traffic(config, G, n, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture of this exact
    workload and launch size (profiles/ncu_traffic.json "r2"); (None, None) when none matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            e = json.load(fh).get("r2", {}).get(f"config{config}:G{G}:n{n}:{kernel}")
        return (e["traffic"], e["source"]) if e else (None, None)
    except Exception:
        return None, None


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


def oracle_run(config, keys, cols, G, K, threads):
    """The oracle on host rows: (status, [outputs], counts or None)."""
    import oracle as O
    if config in ARRAY:
        rc, v = O.dot(cols[0], cols[1], K, threads=threads) if len(cols) == 2 else O.rsum(cols[0], K, threads=threads)
        return rc, [np.array([v])], None
    if config == 4:
        return O.groupby_sum_multi(keys, cols, G, K, proj=1, threads=threads)
    rc, out = O.groupby_sum(keys, cols[0], G, K, threads=threads)
    return rc, [out], None


def cpu_baseline(args, n, G, K):
    """The oracle as it stands, on a bounded sample of the workload (rows
    [0, S) of this rank's shard), all host threads."""
    import oracle as O
    sample = min(n, ORACLE_SAMPLE_ROWS)
    keys, cols = host_rows(args.config, 0, sample, G)
    threads = O.default_threads()
    t0 = time.perf_counter()
    rc, _, _ = oracle_run(args.config, keys, cols, G, K, threads)
    t = time.perf_counter() - t0
    if rc != 0:
        raise SystemExit(f"oracle status {rc}")
    return {"value": sample / t, "unit": "rows/s", "cores": threads, "kind": "oracle",
            "sample": f"rows [0, {sample}) of the workload ({'4 SUM columns + COUNT, ' if args.config == 4 else ''}"
                      f"{threads} host threads)", "seconds": t}


def repo_libs_mapped():
    """Shared objects under the repo root mapped into this process."""
    libs = set()
    try:
        with open("/proc/self/maps") as fh:
            for ln in fh:
                path = ln.split()[-1] if len(ln.split()) >= 6 else ""
                if path.endswith(".so") and path.startswith(ROOT):
                    libs.add(os.path.relpath(path, ROOT))
    except OSError:
        return None
    return sorted(libs)


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands, timed on the host cores
    (rank 0 only; other ranks exit without work).  Each step is a bounded
    sample of the workload -- consecutive row blocks of it -- sized so that all
    K steps together process at most 2^28 rows (2^26 for config 4)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    n, G, K, dt = shape(args)
    steps = max(1, args.steps)
    budget = (1 << 26) if args.config == 4 else (1 << 28)
    sample = max(1 << 12, min(n, budget // steps))
    threads = O.default_threads()
    keys, cols = host_rows(args.config, 0, min(n, sample * steps), G)
    if keys is None:
        keys = np.zeros(cols[0].size, np.int32)  # placeholder for slicing (keyless workloads)
    for _ in range(args.warmup):
        oracle_run(args.config, keys[: 1 << 12], [c[: 1 << 12] for c in cols], G, K, threads)
    times = []
    total_rows = keys.size
    for s in range(steps):
        a = (s * sample) % max(1, total_rows - sample + 1)
        t0 = time.perf_counter()
        rc, _, _ = oracle_run(args.config, keys[a:a + sample], [c[a:a + sample] for c in cols], G, K, threads)
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
        # shared objects of this repo mapped into the arm's process: the oracle
        # only (the arm never imports the product package)
        "repo_libs_mapped": repo_libs_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- one workload: timed steps, per-kernel roofline, baselines, parity ----------

CONFIG2_GROUPS = [16, 1024, 4096, 1 << 16, 1 << 20, 1 << 24]  # sub-results of the default run


def oracle_parity(R, torch, config, keys, cols, host, G, K, outs, counts):
    """Bit comparison of the GPU outputs with the oracle on the SAME input
    bytes (D2H copies of the device rows, or the host rows they came from).
    Full comparison where the oracle finishes in seconds; 258 sampled groups
    recomputed one by one at G > 2^20; config 4 streamed in shards of 2^26
    rows whose oracle states are merged with the oracle's own merge (O3)."""
    import oracle as O
    thr = O.default_threads()
    if config in ARRAY:
        hc = host[1] if host else [c.cpu().numpy() for c in cols]
        rc, ref, _ = oracle_run(config, None, hc, G, K, thr)
        ok = rc == 0 and outs[0].cpu().numpy().tobytes() == ref[0].tobytes()
        return {"vs_oracle": "bit-exact" if ok else "MISMATCH", "rows_compared": int(hc[0].size)}
    if config == 4:
        n = keys.numel()
        p = O.params(O.F64, K)
        states = [[None] * G for _ in range(4)]
        cnt = np.zeros(G, np.int64)
        sh = 1 << 26
        for a in range(0, n, sh):
            b = min(n, a + sh)
            hk = keys[a:b].cpu().numpy()
            hc = [c[a:b].cpu().numpy() for c in cols]
            dp, ch = O.q1_project(hc[1], hc[2], hc[3])
            for j, c in enumerate([hc[0], hc[1], dp, ch]):
                rc, _, st = O.groupby_sum(hk, c, G, K, threads=thr, with_state=True)
                if rc != 0:
                    return {"vs_oracle": f"oracle status {rc}", "rows_compared": n}
                for g in range(G):
                    s_ = O.State(list(st[g, :K]), list(st[g, K:]))
                    if states[j][g] is None:
                        states[j][g] = s_
                    elif O.merge(p, states[j][g], s_) != 0:
                        return {"vs_oracle": "oracle merge error", "rows_compared": n}
            cnt += np.bincount(hk[(hk >= 0) & (hk < G)], minlength=G)
        ok = np.array_equal(counts.cpu().numpy(), cnt)
        for j in range(4):
            ref = np.array([O.finalize(p, states[j][g]) for g in range(G)], np.float64)
            ok = ok and outs[j].cpu().numpy().tobytes() == ref.tobytes()
        return {"vs_oracle": "bit-exact" if ok else "MISMATCH", "groups": G, "rows_compared": n, "columns": 4,
                "counts": True, "oracle_shards": -(-n // sh)}
    hk = host[0] if host else keys.cpu().numpy()
    hv = host[1][0] if host else cols[0].cpu().numpy()
    got = outs[0].cpu().numpy()
    if G <= (1 << 20):
        rc, ref = O.groupby_sum(hk, hv, G, K, threads=thr)
        ok = rc == 0 and got.tobytes() == ref.tobytes()
        return {"vs_oracle": "bit-exact" if ok else "MISMATCH", "groups": G, "rows_compared": int(hk.size)}
    rng = np.random.default_rng(0)
    sel = np.unique(np.concatenate([[0, G - 1], rng.integers(0, G, 256)])).astype(np.int32)
    rc, ref = O.groupby_sum_select(hk, hv, G, K, sel, threads=thr)
    ok = rc == 0 and got[sel].tobytes() == ref.tobytes()
    return {"vs_oracle": "bit-exact" if ok else "MISMATCH", "groups_sampled": int(sel.size),
            "rows_compared": int(hk.size)}


def run_sparse(R, torch, steps, warmup):
    """f1: repro_groupby_sum_sparse (hash table -> sorted dense ids -> dense
    path; blocking) on host-generated int64 keys; parity against the oracle's
    np.unique + O5 on the same rows."""
    from inputs import synth
    n, D, K = SPARSE["n"], SPARSE["distinct"], 3
    seed = synth.SEED_BASE + 7
    hk = synth.keys_sparse(seed, 0, n, D)
    hv = synth.values_signed_mant_exp(synth.SEED_BASE + 1, 0, n)
    keys, vals = torch.from_numpy(hk).cuda(), torch.from_numpy(hv).cuda()
    for _ in range(max(3, warmup)):
        uk, out = R.groupby_sum_sparse(keys, vals, D)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    for _ in range(steps):
        uk, out = R.groupby_sum_sparse(keys, vals, D)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peak, _ = peaks()
    res = {"workload": WORKLOADS[7], "config": 7, "rows_per_gpu": n, "distinct_keys": int(uk.numel()), "fold": K,
           "dtype": "f64", "ms_per_step": ms, "value": n / (ms * 1e-3), "unit": "rows/s",
           "step_hbm_gbs": n * 16 / (ms * 1e-3) / 1e9, "step_roofline_frac": n * 16 / (ms * 1e-3) / 1e9 / peak,
           "note": "blocking call (the distinct count is read back to size the dense pass); the step reads "
                   "16 B/row of input (int64 key + fp64 value)"}
    import oracle as O
    t0 = time.perf_counter()
    rc, ruk, rout = O.groupby_sum_sparse(hk, hv, K)
    ok = rc == 0 and np.array_equal(uk.cpu().numpy(), ruk) and out.cpu().numpy().tobytes() == rout.tobytes()
    res["parity"] = {"vs_oracle": "bit-exact" if ok else "MISMATCH", "groups": int(ruk.size), "rows_compared": n,
                     "seconds": time.perf_counter() - t0}
    del keys, vals
    torch.cuda.empty_cache()
    return res


def run_workload(R, torch, args, config, n, G, K, dts, world, rank, local, steps, warmup, *, parity=True,
                 atomic=True, headline=False):
    """Time the whole hot path on one workload; returns the result dict."""
    import torch.distributed as dist
    from paper_1802_09883_b200 import dist as rdist
    dt = R.F64 if dts == "f64" else R.F32
    vsz = 8 if dt == R.F64 else 4
    multi = config == 4
    array = config in ARRAY
    ncol = 4 if multi else (2 if array and ARRAY[config]["dot"] else 1)
    row_bytes = (0 if array else 4) + ncol * vsz
    host = None
    if config == 3:  # transcendental values: generated on the host, uploaded
        hk, hc = host_rows(config, rank * n, n, G)
        host = (hk, hc)
        keys, cols = torch.from_numpy(hk).cuda(), [torch.from_numpy(c).cuda() for c in hc]
    else:
        keys, cols = device_rows(R, torch, config, rank * n, n, G)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    counts = None
    if array:
        outs = [torch.empty(1, dtype=cols[0].dtype, device="cuda")]
        ws = R.make_dot_workspace(K, dt)
        ycol = cols[1] if ncol == 2 else None
    elif multi:
        outs = [torch.empty(G, dtype=torch.float64, device="cuda") for _ in range(4)]
        counts = torch.empty(G, dtype=torch.int64, device="cuda")
        ws = R.make_multi_workspace(n, G, 4, 1, K, dt)
    else:
        outs = [torch.empty(G, dtype=cols[0].dtype, device="cuda")]
        ws = R.make_workspace(n, G, K, dt)
    nvls = None
    if world > 1 and not multi and not array and G < 4096:  # NVSwitch multicast table all-reduce when available
        nvls = rdist.NvlsWorkspace.create(ws.numel())
        if nvls is not None:
            ws = nvls.buf
    acc = None

    def step():
        if array:
            if world == 1:
                R.dot_async(cols[0], ycol, K, outs[0], ws, status, stream)
            else:  # deposit, all-reduce the integer slot table, read out on every rank
                rdist.dot_dist(R, cols[0], ycol, K, outs[0], ws, status, stream=stream)
            return
        if multi:
            if world == 1:
                R.groupby_sum_multi_async(keys, cols, G, K, 1, outs, counts, ws, status, stream)
            else:  # deposit, all-reduce the integer slot tables, read out on every rank
                rdist.groupby_sum_multi_dist(R, keys, cols, G, K, 1, outs, counts, ws, status, stream=stream)
            return
        if world == 1:
            R.groupby_sum_async(keys, cols[0], G, K, outs[0], ws, status, stream)
            return
        # stream-ordered split form: deposit into the slot table, integer
        # collectives on the same stream (OR/MAX/SUM; G >= 4096: reduce-scatter
        # by group range + all-gather of the outputs), read-out -- no host sync
        rdist.groupby_sum_dist(R, keys, cols[0], G, K, outs[0], ws, status, stream=stream, nvls=nvls)

    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    if int(status.item()) != 0:
        raise SystemExit(f"device status {status.item()} in warm-up ({WORKLOADS.get(config)}, G={G})")

    def timed_region(per_kernel):
        R.timing_enable(per_kernel)
        R.timing_collect()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for _ in range(steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        R.timing_enable(False)
        pk = R.timing_collect()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, pk, clk.result()

    # region A: the step as a user runs it (no per-kernel events) -> value
    ms, _, clocks = timed_region(False)
    st_a = int(status.item())
    # region B: the same steps with every library kernel bracketed by events
    # on its stream -> per-kernel times and the dominant kernel's roofline
    ms_b, per_kernel, _ = timed_region(True)
    st_b = int(status.item())
    ms_per_step = ms / steps
    rows_total = n * world
    value = rows_total / (ms_per_step * 1e-3)
    peak, peak_src = peaks()
    dom = max(per_kernel.items(), key=lambda kv: kv[1][1]) if per_kernel else None
    roof = None
    if dom:
        name, (cnt, kms) = dom
        avg_ms = kms / cnt
        alg_bytes = n * row_bytes  # the kernel's algorithmic input bytes per launch
        achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
        traffic, traffic_src = ncu_traffic(config, G, n, name)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": name, "kernel_ms": avg_ms,
                "kernel_share_of_step": kms / ms_b if ms_b else None, "alg_bytes_per_launch": alg_bytes,
                "alg_bytes_per_row": row_bytes, "peak_source": peak_src,
                "traffic_note": ("dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full capture "
                                 "of this workload: " + traffic_src) if traffic_src else
                "no ncu --set full capture of this kernel at this launch size (profiles/r2_*_ncu_full.txt)"}
    if roof is not None:
        # FP side of the roofline: 3K - 2 correctly rounded
        # adds per deposited value at the MEASURED add rate of this GPU
        rate = fp_add_rate(R, dt)
        fp_adds = n * ncol * (3 * K - 2)
        t_hbm = alg_bytes / (peak * 1e9)
        t_fp = fp_adds / rate
        roof.update({"fp_add_rate_measured": rate, "fp_adds_per_launch": fp_adds, "hbm_time_ms": t_hbm * 1e3,
                     "fp_time_ms": t_fp * 1e3, "fp_pipe_frac": t_fp / (roof["kernel_ms"] * 1e-3),
                     "roofline_time_ms": max(t_hbm, t_fp) * 1e3})
        if t_fp > t_hbm:
            roof["bound"] = "alu"
    step_bytes = n * row_bytes + G * vsz * (5 if multi else 1)
    res = {
        "workload": WORKLOADS.get(config), "config": config, "rows_per_gpu": n, "n_groups": G, "fold": K,
        "dtype": dts, "ms_per_step": ms_per_step, "value": value, "unit": "rows/s",
        "step_hbm_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
        "step_roofline_frac": (step_bytes / (ms_per_step * 1e-3) / 1e9) / peak,
        "roofline": roof, "per_kernel_ms": {k: v[1] / v[0] for k, v in per_kernel.items()},
        "gpu_launches": sum(c for c, _ in per_kernel.values()), "path": R.last_path(), "clocks": clocks,
        "device_status_after_timed_steps": st_a if st_a else st_b,
    }
    if st_a or st_b:
        res["rejected"] = f"device status {st_a or st_b} during the timed steps"

    # non-reproducible atomicAdd GroupBy on the same GPU and the same rows:
    # the fastest of the five variants (global RED per row, shared-memory
    # table, register partials for <= 16 groups, warp aggregation of equal
    # keys, heavy hitters privatised per block)
    if atomic and world == 1 and not multi and not array:
        best = None
        for variant in (0, 1, 2, 3, 4):
            try:
                for _ in range(3):
                    R.baseline_atomic_sum(keys, cols[0], G, variant=variant, stream=stream)
                torch.cuda.synchronize()
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                bsteps = max(5, steps // 2)
                b0.record(stream)
                for _ in range(bsteps):
                    R.baseline_atomic_sum(keys, cols[0], G, variant=variant, stream=stream)
                b1.record(stream)
                torch.cuda.synchronize()
                bms = b0.elapsed_time(b1) / bsteps
                if best is None or bms < best[1]:
                    best = (variant, bms)
            except R.ReproError:
                continue
        if best:
            names = ["global_atomicAdd", "smem_privatised_atomicAdd", "register_partials_atomicAdd",
                     "warp_aggregated_atomicAdd", "heavy_hitters_privatised_atomicAdd"]
            res["baseline_atomic"] = {"variant": names[best[0]], "ms_per_step": best[1],
                                      "rows_per_s": n / (best[1] * 1e-3),
                                      "slowdown_repro_vs_atomic": ms_per_step / best[1]}

    if headline and not args.no_e2e and world == 1 and not multi and not array:
        kp = keys.cpu().pin_memory()
        vp = cols[0].cpu().pin_memory()
        R.groupby_sum_host(kp, vp, G, K)
        e2e_steps = max(3, min(steps, 10))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r_ = R.groupby_sum_host(kp, vp, G, K)
        et = (time.perf_counter() - t0) / e2e_steps
        kd2, vd2 = torch.empty_like(keys), torch.empty_like(cols[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            kd2.copy_(kp, non_blocking=True)
            vd2.copy_(vp, non_blocking=True)
        torch.cuda.synchronize()
        h2d = 3 * n * row_bytes / (time.perf_counter() - t0) / 1e9
        del kd2, vd2
        res["e2e"] = {"value": n / et, "unit": "rows/s", "h2d_bytes_per_step": n * row_bytes,
                      "d2h_bytes_per_step": G * vsz, "ms_per_step": et * 1e3, "steps": e2e_steps,
                      "h2d_copy_gbs": h2d, "e2e_gbs": n * row_bytes / et / 1e9,
                      "bit_identical_to_device_path": bool(torch.equal(r_, outs[0].cpu()))}
        del kp, vp

    if parity and rank == 0 and world == 1 and not args.no_parity:
        t0 = time.perf_counter()
        res["parity"] = oracle_parity(R, torch, config, keys, cols, host, G, K, outs, counts)
        res["parity"]["seconds"] = time.perf_counter() - t0
    del keys, cols, ws, outs, acc
    torch.cuda.empty_cache()
    return res


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
    head = run_workload(R, torch, args, args.config, n, G, K, dts, world, rank, local, args.steps, args.warmup,
                        headline=True)
    line = {
        "metric": METRIC, "value": head["value"], "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dts, "data": "synthetic",
        "config": {"workload": WORKLOADS.get(args.config), "rows_per_gpu": n, "n_groups": G, "fold": K,
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": f"inputs {n * (head['roofline'] or {}).get('alg_bytes_per_row', 12) / 1e9:.2f} GB/GPU "
                         f"> 126 MB L2 (no flush needed)"},
    }
    for k in ("step_hbm_gbs", "step_roofline_frac", "roofline", "per_kernel_ms", "gpu_launches", "path", "clocks",
              "baseline_atomic", "e2e", "parity", "device_status_after_timed_steps", "rejected"):
        if k in head:
            line[k] = head[k]

    # the other BASELINE configs, measured in the same process (N = 1, default run)
    if world == 1 and not args.no_configs and args.config == 1 and args.rows is None:
        subs = {}
        for g in CONFIG2_GROUPS:
            subs[f"config2_G{g}"] = run_workload(R, torch, args, 2, 1 << 28, g, 3, "f64", world, rank, local,
                                                 args.steps, args.warmup)
        subs["config3"] = run_workload(R, torch, args, 3, 1 << 28, 1 << 20, 2, "f32", world, rank, local,
                                       args.steps, args.warmup)
        subs["config4"] = run_workload(R, torch, args, 4, 1 << 30, 4, 3, "f64", world, rank, local,
                                       max(3, args.steps // 4), args.warmup)
        subs["f1_sparse"] = run_sparse(R, torch, max(3, args.steps // 4), args.warmup)
        line["configs"] = subs

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, n, G, K)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
