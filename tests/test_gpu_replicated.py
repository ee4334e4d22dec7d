"""GPU parity of the sweep's replicated-read form (k_sweep_hot<REP>, k_sweep.cu):
for plans of a few partitions each row chunk is read by one block per
partition, each depositing only its own partition's rows on chip (no scatter).
The form is selected by REPRO_SWEEP_REP_MAXP (read at every call); results must
be bit-identical to the oracle (Alg. 1 / Eq. 1) and to the
scatter form, whatever the knob."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402  (test infrastructure)


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


@pytest.fixture(params=["0", "2", "4"])
def maxp(request):
    old = os.environ.get("REPRO_SWEEP_REP_MAXP")
    os.environ["REPRO_SWEEP_REP_MAXP"] = request.param
    yield int(request.param)
    if old is None:
        os.environ.pop("REPRO_SWEEP_REP_MAXP", None)
    else:
        os.environ["REPRO_SWEEP_REP_MAXP"] = old


def values(rng, n, dtype, lo, hi):
    e = rng.integers(lo, hi + 1, n)
    return (rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1.0, 1.0], n)).astype(dtype)


def check(R, keys, vals, G, K):
    out = R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, K)
    torch.cuda.synchronize()
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    got = out.cpu().numpy()
    iu = np.uint64 if got.dtype == np.float64 else np.uint32
    bad = np.nonzero(got.view(iu) != ref.view(iu))[0]
    assert bad.size == 0, f"{bad.size} groups differ, first {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"


@pytest.mark.parametrize("dtype,K,G", [(np.float64, 3, 8192), (np.float64, 3, 7001), (np.float64, 3, 12288),
                                       (np.float64, 3, 16384), (np.float64, 2, 20000), (np.float32, 2, 30000),
                                       (np.float32, 3, 17000)])
@pytest.mark.parametrize("n", [(1 << 21) + 5, 1000, 3])
def test_replicated_read_parity(R, maxp, dtype, K, G, n):
    rng = np.random.default_rng(G + n + K)
    keys = rng.integers(0, G, n).astype(np.int32)
    lo, hi = ((-30, 60) if dtype == np.float64 else (-20, 25))  # window tops 0 .. 2: band mode, rows outside the band
    check(R, keys, values(rng, n, dtype, lo, hi), G, K)


def test_replicated_read_skewed_and_untouched_partitions(R, maxp):
    # every row in the last partition but three: the other blocks see only foreign rows
    rng = np.random.default_rng(77)
    G, n = 12288, (1 << 20) + 1
    keys = rng.integers(8192, G, n).astype(np.int32)
    keys[[5, n // 2, n - 1]] = [0, 4097, 8191]
    check(R, keys, values(rng, n, np.float64, -20, 20), G, 3)


@pytest.mark.parametrize("bad", [-1, "G", "big"])
def test_replicated_read_bad_key(R, maxp, bad):
    rng = np.random.default_rng(5)
    G, n = 8192, (1 << 20) + 7
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = values(rng, n, np.float64, -20, 20)
    keys[n - 6] = {-1: -1, "G": G, "big": 2 ** 31 - 1}[bad]
    assert O.groupby_sum(keys, vals, G, 3)[0] == O.EKEY
    with pytest.raises(R.ReproError) as ei:
        R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, 3)
    torch.cuda.synchronize()
    assert ei.value.status == O.EKEY


def test_replicated_read_nan_is_edom(R, maxp):
    rng = np.random.default_rng(6)
    G, n = 8192, (1 << 20) + 2
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = values(rng, n, np.float64, -20, 20)
    vals[n // 3] = np.nan
    assert O.groupby_sum(keys, vals, G, 3)[0] == O.EDOM
    with pytest.raises(R.ReproError) as ei:
        R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, 3)
    torch.cuda.synchronize()
    assert ei.value.status == O.EDOM


def test_replicated_read_unaligned(R, maxp):
    rng = np.random.default_rng(8)
    G, n, off = 8192, (1 << 20) + 3, 1
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = values(rng, n, np.float64, -20, 20)
    kt = torch.zeros(n + off, dtype=torch.int32, device="cuda")
    vt = torch.zeros(n + off, dtype=torch.float64, device="cuda")
    kt[off:] = torch.from_numpy(keys).cuda()
    vt[off:] = torch.from_numpy(vals).cuda()
    out = R.groupby_sum(kt[off:], vt[off:], G, 3)
    torch.cuda.synchronize()
    rc, ref = O.groupby_sum(keys, vals, G, 3)
    assert rc == O.OK
    assert out.cpu().numpy().view(np.uint64).tobytes() == ref.view(np.uint64).tobytes()


def test_replicated_read_host_entry_and_chunked_handle(R, maxp):
    # the host entry point (H2D chunks pipelined with deposits) and the handle API (deposits merged into a
    # canonical state) go through the same form; state and sums equal the oracle's
    rng = np.random.default_rng(9)
    G, n = 8000, (1 << 21) + 11
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = values(rng, n, np.float64, -30, 60)
    rc, ref, st = O.groupby_sum(keys, vals, G, 3, with_state=True)
    assert rc == O.OK
    got = R.groupby_sum_host(torch.from_numpy(keys).pin_memory(), torch.from_numpy(vals).pin_memory(), G, 3).numpy()
    assert got.view(np.uint64).tobytes() == ref.view(np.uint64).tobytes()
    a = R.Accumulator(G, 3, R.F64)
    for c0, c1 in ((0, 5), (5, 1 << 20), (1 << 20, n)):
        a.deposit(torch.from_numpy(keys[c0:c1]).cuda(), torch.from_numpy(vals[c0:c1]).cuda())
    assert a.finalize().cpu().numpy().view(np.uint64).tobytes() == ref.view(np.uint64).tobytes()
    assert a.export().cpu().numpy().reshape(G, 6).tobytes() == st.tobytes()
