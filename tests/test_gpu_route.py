"""GPU parity of the routed one-pass kernel (csrc/k_route.cu): every SM
streams its rows once and sends each row to the SM whose shared-memory table
owns the row's group (g mod Q) through an L2 ring buffer; heavy keys stay with
their producer.  PartitionAndAggregate (Alg. 4) with the
partitions streamed instead of written out.  Checked bit for bit against the
oracle (Alg. 1 / Eq. 1) and against the two-pass sweep
(route off), with

  * group counts from just above one SM's table to ~1M (Q = 2 .. 148),
  * uniform and Zipf keys (heavy keys deposited by the producers),
  * values whose window tops fall inside the band, below and above it
    (rows deposited one by one into the slot table),
  * inputs that wrap every ring many times, tiny inputs (most producers
    empty), ragged lengths and unaligned row arrays,
  * error rows (EKEY > EDOM > ERANGE precedence),
  * K = 1 .. 4, binary64 and binary32."""
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
    R.set_route_mode(1)  # opt-in path
    yield R
    R.set_route_mode(0)


def zipf_keys(rng, n, G, s=1.1):
    p = np.arange(1, G + 1, dtype=np.float64) ** -s
    cdf = np.cumsum(p / p.sum())
    return np.minimum(np.searchsorted(cdf, rng.random(n)), G - 1).astype(np.int32)


def values(rng, n, dtype, lo, hi):
    """|v| = (1 + mant) 2^e, e uniform in [lo, hi], random sign."""
    e = rng.integers(lo, hi + 1, n)
    return (rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1.0, 1.0], n)).astype(dtype)


def gpu(R, keys, vals, G, K, offset=0):
    """GroupBy on the device; offset > 0 shifts both row arrays by that many
    elements (unaligned 16-byte loads)."""
    if offset:
        kt = torch.zeros(len(keys) + offset, dtype=torch.int32, device="cuda")
        vt = torch.zeros(len(vals) + offset, dtype=torch.from_numpy(vals).dtype, device="cuda")
        kt[offset:] = torch.from_numpy(keys).cuda()
        vt[offset:] = torch.from_numpy(vals).cuda()
        k, v = kt[offset:], vt[offset:]
    else:
        k, v = torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda()
    R.timing_enable(True)
    try:
        out = R.groupby_sum(k, v, G, K)
        torch.cuda.synchronize()
        names = R.timing_collect()
    finally:
        R.timing_enable(False)
    return out.cpu().numpy(), names


def check(R, keys, vals, G, K, routed=True, offset=0):
    got, names = gpu(R, keys, vals, G, K, offset)
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    iu = np.uint64 if got.dtype == np.float64 else np.uint32
    bad = np.nonzero(got.view(iu) != ref.view(iu))[0]
    assert bad.size == 0, f"{bad.size} groups differ, first {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"
    assert R.last_path() == 1
    assert ("route" in names) == routed, names
    return got


# binary64: window tops 0 / 1 / 2 for |v| < 2^-13 / < 2^27 / < 2^67;
# binary32: 0 / 1 / 2 for |v| < 2^-6 / < 2^12 / < 2^30
SPANS = {np.float64: [(-30, 20), (-20, 40), (-30, 60)], np.float32: [(-10, 10), (-12, 16), (-20, 25)]}


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2)])
@pytest.mark.parametrize("G", [7000, 20011, 1 << 16, 300001, 1 << 20])
def test_route_uniform_keys(R, dtype, K, G):
    if G <= R.onchip_max_groups(K, 1 if dtype == np.float64 else 0):
        pytest.skip("on-chip table path")
    rng = np.random.default_rng(G + K)
    n = (1 << 21) + 7
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = (2.0 * rng.random(n) - 1.0).astype(dtype)  # config-2 values
    check(R, keys, vals, G, K)


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2)])
@pytest.mark.parametrize("span", [0, 1, 2])
def test_route_zipf_heavy_and_window_spans(R, dtype, K, span):
    rng = np.random.default_rng(100 + span + K)
    G, n = 1 << 18, (1 << 21) + 3
    lo, hi = SPANS[dtype][span]
    check(R, zipf_keys(rng, n, G), values(rng, n, dtype, lo, hi), G, K)


def test_route_config3_shape(R):
    # Zipf(1.1) over 2^20 keys, binary32 normal * 2^e, K = 2 (BASELINE config 3 at 2^23 rows)
    rng = np.random.default_rng(3)
    G, n = 1 << 20, (1 << 23) + 1
    keys = zipf_keys(rng, n, G)
    vals = (rng.standard_normal(n) * np.exp2(rng.integers(-10, 11, n))).astype(np.float32)
    check(R, keys, vals, G, 2)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_route_every_fold(R, dtype, K):
    rng = np.random.default_rng(40 + K)
    G, n = 50000, (1 << 20) + 2
    check(R, rng.integers(0, G, n, dtype=np.int32), values(rng, n, dtype, *SPANS[dtype][1]), G, K)


def test_route_many_ring_laps(R):
    # 2^24 rows over ~148 consumers: ~14 laps of every 8192-row ring
    rng = np.random.default_rng(9)
    G, n = 9000, 1 << 24
    check(R, rng.integers(0, G, n, dtype=np.int32), (2.0 * rng.random(n) - 1.0), G, 3)


@pytest.mark.parametrize("n", [1, 5, 300, 4097])
def test_route_tiny_inputs(R, n):
    rng = np.random.default_rng(n)
    G = 100000
    check(R, rng.integers(0, G, n, dtype=np.int32), values(rng, n, np.float64, -20, 20), G, 3)


def test_route_empty_input(R):
    got, _ = gpu(R, np.zeros(0, np.int32), np.zeros(0, np.float64), 100000, 3)
    assert not np.any(got.view(np.uint64))


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_route_unaligned_rows(R, offset):
    rng = np.random.default_rng(offset)
    G, n = 30000, (1 << 20) + 11
    check(R, rng.integers(0, G, n, dtype=np.int32), values(rng, n, np.float64, -20, 20), G, 3, offset=offset)


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2)])
def test_route_equals_sweep(R, dtype, K):
    rng = np.random.default_rng(77)
    G, n = 1 << 17, (1 << 21) + 1
    keys = zipf_keys(rng, n, G)
    vals = values(rng, n, dtype, *SPANS[dtype][2])
    a = check(R, keys, vals, G, K, routed=True)
    R.set_route_mode(0)
    try:
        b = check(R, keys, vals, G, K, routed=False)
    finally:
        R.set_route_mode(1)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("bad", ["key", "nan", "huge", "all"])
def test_route_error_rows(R, bad):
    rng = np.random.default_rng(5)
    G, n = 40000, (1 << 20) + 1
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = values(rng, n, np.float64, -20, 20)
    if bad in ("key", "all"):
        keys[n - 3] = G
    if bad in ("nan", "all"):
        vals[n // 2] = np.nan
    if bad in ("huge", "all"):
        vals[17] = 2.0 ** 990
    want = {"key": O.EKEY, "nan": O.EDOM, "huge": O.ERANGE, "all": O.EKEY}[bad]
    rc, _ = O.groupby_sum(keys, vals, G, 3)
    assert rc == want
    with pytest.raises(R.ReproError) as ei:
        R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, 3)
    torch.cuda.synchronize()
    assert ei.value.status == want
