"""Multi-rank exchange on CPU: world_size 2 over gloo.

`paper_1802_09883_b200.dist.allreduce_state` is the host logic the bench runs
over NCCL.  Here each rank's accumulator is a test double backed by the CPU
oracle (state of the rank's shard) that implements the same three calls as
the CUDA Accumulator: top_levels / window_export / window_import.  The
combined state must equal the oracle over all rows, bit for bit, on every rank
and for any sharding.
"""
import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import exact_ref as X
import oracle as O

FMT = {O.F64: (52, 40), O.F32: (23, 18)}


class OracleAccumulator:
    """Test double: the oracle's state of a shard, in integer window form."""

    def __init__(self, keys, vals, G, K):
        self.G, self.K = G, K
        self.n_groups, self.fold = G, K
        self.dtype = O.F64 if vals.dtype == np.float64 else O.F32
        rc, _, st = O.groupby_sum(keys, vals, G, K, threads=1, with_state=True)
        assert rc == O.OK
        m, W = FMT[self.dtype]
        self.k = np.zeros(G, np.int64)
        self.T = [[0] * K for _ in range(G)]
        for g in range(G):
            S, C = st[g, :K], st[g, K:]
            e0 = int(np.frexp(S[0])[1]) - 1
            self.k[g] = e0 // W
            for l in range(K):
                e = e0 - W * l
                D = Fraction(float(S[l])) - Fraction(3, 2) * Fraction(2) ** e
                u = Fraction(2) ** (e - m)
                self.T[g][l] = int(D / u) + int(C[l]) * (1 << (m - 2))

    def top_levels(self):
        return torch.tensor(self.k, dtype=torch.int32)

    def window_export(self, k_global):
        kg = k_global.numpy()
        out = np.zeros((self.G, self.K, 2), np.int64)
        for g in range(self.G):
            sh = int(kg[g]) - int(self.k[g])
            assert sh >= 0
            T = [0] * sh + self.T[g][: self.K - sh] if sh < self.K else [0] * self.K
            for l in range(self.K):
                out[g, l, 0] = T[l] & 0xFFFFFFFF
                out[g, l, 1] = T[l] >> 32
        return torch.from_numpy(out.reshape(-1))

    def window_import(self, k_global, limbs, g0=0, count=None):
        count = self.G - g0 if count is None else count
        L = limbs.numpy().reshape(count, self.K, 2)
        kg = k_global.numpy().astype(np.int64)
        for i in range(count):
            self.k[g0 + i] = kg[i]
            self.T[g0 + i] = [(int(L[i, l, 1]) << 32) + int(L[i, l, 0]) for l in range(self.K)]
        return self

    def finalize(self):
        bits = 64 if self.dtype == O.F64 else 32
        return np.array([X.finalize_closed_form(int(self.k[g]), self.T[g], bits) for g in range(self.G)],
                        dtype=np.float64 if bits == 64 else np.float32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys, vals, G, K, shard, q, exchange="allreduce"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_09883_b200 import dist as rdist
        if shard == "contiguous":
            r0, r1 = rdist.shard_rows(keys.size, world, rank)
            k, v = keys[r0:r1], vals[r0:r1]
        else:
            k, v = keys[rank::world], vals[rank::world]
        acc = OracleAccumulator(k, v, G, K)
        if exchange == "reduce_scatter":
            out = torch.empty(G, dtype=torch.float64 if vals.dtype == np.float64 else torch.float32)
            rdist.reduce_scatter_finalize(acc, out)
            q.put((rank, out.numpy().tobytes()))
        else:
            rdist.allreduce_state(acc)
            q.put((rank, acc.finalize().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,K,shard,exchange,world,G", [
    (np.float64, 3, "contiguous", "allreduce", 2, 12), (np.float64, 2, "strided", "allreduce", 2, 12),
    (np.float32, 2, "contiguous", "allreduce", 2, 12),
    (np.float64, 3, "contiguous", "reduce_scatter", 2, 13), (np.float32, 2, "strided", "reduce_scatter", 3, 7),
    (np.float64, 2, "contiguous", "reduce_scatter", 3, 2)])
def test_two_rank_exchange_equals_single_oracle(dtype, K, shard, exchange, world, G):
    rng = np.random.default_rng(11)
    n = 6000
    keys = rng.integers(0, G, n, dtype=np.int32)
    e = rng.integers(-30, 31, n)
    vals = (rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1, 1], n)).astype(dtype)
    vals[:7] *= 2.0 ** 50 if dtype == np.float64 else 2.0 ** 20  # rank 0 needs higher windows
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, vals, G, K, shard, q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res[r] == ref.tobytes() for r in range(world))


def test_shard_rows_cover_everything():
    from paper_1802_09883_b200 import dist as rdist
    for n in (0, 1, 7, 1000):
        for world in (1, 2, 3, 8):
            spans = [rdist.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


# ---- slot-table exchange of the fused multi-column pass -------------------

NS = {O.F64: 25, O.F32: 7}  # KMAX per dtype; a table row holds KMAX + K absolute-level slots


def _slot_table(acc):
    """The absolute-level slot table layout of the on-chip kernels (k_fold):
    slots[g][level + K - 1] = (sum of low 32-bit parts, sum of high parts) of
    the level sum at that absolute level, kglob[g] = window top."""
    G, K = acc.G, acc.K
    ns = NS[acc.dtype] + K
    slots = np.zeros((G, ns, 2), np.int64)
    for g in range(G):
        k = int(acc.k[g])
        for l in range(K):
            T = acc.T[g][l]
            slots[g, k - l + K - 1, 0] = T & 0xFFFFFFFF
            slots[g, k - l + K - 1, 1] = T >> 32
    return torch.tensor(acc.k, dtype=torch.int32), torch.from_numpy(slots.reshape(-1))


def _table_worker(rank, world, port, keys, vals, G, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_09883_b200 import dist as rdist
        r0, r1 = rdist.shard_rows(keys.size, world, rank)
        acc = OracleAccumulator(keys[r0:r1], vals[r0:r1], G, K)
        kglob, slots = _slot_table(acc)
        flags = torch.tensor([1 << rank], dtype=torch.int32)  # each rank raises another status bit
        rdist.allreduce_table(flags, kglob, slots)
        # read the summed table under the global tops (what k_fold does)
        ns = NS[acc.dtype] + K
        S = slots.numpy().reshape(G, ns, 2)
        acc.k = kglob.numpy().astype(np.int64)
        acc.T = [[(int(S[g, int(acc.k[g]) - l + K - 1, 1]) << 32) + int(S[g, int(acc.k[g]) - l + K - 1, 0])
                  for l in range(K)] for g in range(G)]
        q.put((rank, int(flags.item()), acc.finalize().tobytes()))
    finally:
        dist.destroy_process_group()


def test_two_rank_slot_table_exchange_equals_single_oracle():
    rng = np.random.default_rng(21)
    n, G, K = 5000, 9, 3
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-60, 60, n))
    vals[-5:] *= 2.0 ** 70  # only rank 1 sees the highest windows
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_table_worker, args=(r, 2, port, keys, vals, G, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (f, b) for r, f, b in (q.get(timeout=120) for _ in range(2))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0] == 3  # status bits OR-ed
    assert res[0][1] == res[1][1] == ref.tobytes()


# ---- stream-ordered split form of the single-column GroupBy ----------------

class FakeR:
    """Test double of the binding's split-form calls (groupby_deposit_async,
    groupby_table_views, groupby_finish_async, groupby_window_limbs_async,
    groupby_finish_limbs_async) over CPU tensors: the deposit is the oracle's
    state of the rank's rows laid out as the absolute-level slot table; the
    read-outs are the exact-rational closed form of Eq. 1.  The workspace is a
    dict of the three table tensors."""
    F64, F32 = O.F64, O.F32

    @staticmethod
    def make_ws(G, K, dt):
        ns = NS[dt] + K
        return {"flags": torch.zeros(1, dtype=torch.int32), "kglob": torch.zeros(G, dtype=torch.int32),
                "slots": torch.zeros(G * ns * 2, dtype=torch.int64), "dt": dt}

    @staticmethod
    def groupby_deposit_async(keys, vals, G, K, ws, stream=None):
        k, v = keys.numpy(), vals.numpy()
        bad = (k < 0) | (k >= G)
        ws["flags"][0] = 1 if bad.any() else 0  # EKEY bit; the rows with bad keys deposit nothing
        acc = OracleAccumulator(k[~bad], v[~bad], G, K)
        kg, slots = _slot_table(acc)
        ws["kglob"].copy_(kg)
        ws["slots"].copy_(slots)

    @staticmethod
    def groupby_table_views(ws, n, G, K, dt):
        return ws["flags"], ws["kglob"], ws["slots"]

    @staticmethod
    def _read(ws, G, K, g):
        ns = NS[ws["dt"]] + K
        S = ws["slots"].numpy().reshape(G, ns, 2)
        k = int(ws["kglob"][g])
        return k, [(int(S[g, k - l + K - 1, 1]) << 32) + int(S[g, k - l + K - 1, 0]) for l in range(K)]

    @staticmethod
    def _status(ws):
        f = int(ws["flags"][0])
        return -2 if f & 1 else -3 if f & 2 else -4 if f & 4 else 0

    @staticmethod
    def groupby_finish_async(n, G, K, dt, out, ws, status, stream=None):
        bits = 64 if dt == O.F64 else 32
        for g in range(G):
            k, T = FakeR._read(ws, G, K, g)
            out[g] = X.finalize_closed_form(k, T, bits)
        status[0] = FakeR._status(ws)

    @staticmethod
    def groupby_window_limbs_async(n, G, K, dt, kglob, limbs, ws, stream=None):
        ns = NS[dt] + K
        S = ws["slots"].numpy().reshape(G, ns, 2)
        L = limbs[: G * K * 2].view(G, K, 2)
        for g in range(G):
            k = int(kglob[g])
            for l in range(K):
                L[g, l, 0] = int(S[g, k - l + K - 1, 0])
                L[g, l, 1] = int(S[g, k - l + K - 1, 1])

    @staticmethod
    def groupby_finish_limbs_async(n, G, K, dt, g0, cnt, k_range, limbs_range, out_range, ws, status, stream=None):
        bits = 64 if dt == O.F64 else 32
        L = limbs_range.view(cnt, K, 2)
        for i in range(cnt):
            T = [(int(L[i, l, 1]) << 32) + int(L[i, l, 0]) for l in range(K)]
            out_range[i] = X.finalize_closed_form(int(k_range[i]), T, bits)
        status[0] = FakeR._status(ws)


def _split_worker(rank, world, port, keys, vals, G, K, rs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_09883_b200 import dist as rdist
        r0, r1 = rdist.shard_rows(keys.size, world, rank)
        dt = O.F64 if vals.dtype == np.float64 else O.F32
        ws = FakeR.make_ws(G, K, dt)
        out = torch.empty(G, dtype=torch.float64 if dt == O.F64 else torch.float32)
        status = torch.zeros(1, dtype=torch.int32)
        rdist.groupby_sum_dist(FakeR, torch.from_numpy(keys[r0:r1]), torch.from_numpy(vals[r0:r1]), G, K, out, ws,
                               status, reduce_scatter=rs)
        q.put((rank, int(status.item()), out.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,K,G,world,rs,badkey", [
    (np.float64, 3, 11, 2, False, False), (np.float64, 3, 11, 2, True, False), (np.float32, 2, 7, 3, True, False),
    (np.float64, 2, 5, 3, False, False), (np.float64, 3, 9, 2, True, True)])
def test_split_form_exchange_equals_single_oracle(dtype, K, G, world, rs, badkey):
    rng = np.random.default_rng(31 + G)
    n = 4000
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-40, 40, n))).astype(dtype)
    vals[-3:] *= 2.0 ** 60 if dtype == np.float64 else 2.0 ** 20  # only the last rank sees the top windows
    if badkey:
        keys[5] = G + 2  # rank 0's rows only: every rank must report EKEY
    rc, ref = O.groupby_sum(keys, vals, G, K)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, keys, vals, G, K, rs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (s, b) for r, s, b in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if badkey:
        assert rc == O.EKEY and all(res[r][0] == O.EKEY for r in range(world))
    else:
        assert rc == O.OK and all(res[r] == (0, ref.tobytes()) for r in range(world))
