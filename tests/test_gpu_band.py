"""GPU parity of the table kernels' band mode (table_core.cuh, Table with XB =
1): blocks whose groups do not share one window top after the first tile
stream with every counter at window kuni spanning kuni .. kuni - K, each row
deposited at its own window.  Exercised on the on-chip table (k_table), the
partitioned sweep's accumulate and hot-partition passes, with

  * skewed keys (Zipf over G: most groups untouched in the first tile),
  * values whose window tops spread over {0, 1, 2} (rows in the band, above
    it and below it, which go straight to the slot table),
  * a late switch from band mode to the uniform mode (every group reaching
    the band top),

all bit for bit against the oracle (Alg. 1 / Eq. 1)."""
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


def zipf_keys(rng, n, G, s=1.1):
    p = np.arange(1, G + 1, dtype=np.float64) ** -s
    cdf = np.cumsum(p / p.sum())
    return np.minimum(np.searchsorted(cdf, rng.random(n)), G - 1).astype(np.int32)


def values(rng, n, dtype, lo, hi):
    """|v| = (1 + mant) 2^e, e uniform in [lo, hi], random sign."""
    e = rng.integers(lo, hi + 1, n)
    return (rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1.0, 1.0], n)).astype(dtype)


def run(R, keys, vals, G, K):
    out = R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, K)
    torch.cuda.synchronize()
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    got = out.cpu().numpy()
    iu = np.uint64 if got.dtype == np.float64 else np.uint32
    bad = np.nonzero(got.view(iu) != ref.view(iu))[0]
    assert bad.size == 0, f"{bad.size} groups differ, first {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"


# binary64: window tops 0 / 1 / 2 for |v| < 2^-13 / < 2^27 / < 2^67;
# binary32: 0 / 1 / 2 for |v| < 2^-6 / < 2^12 / < 2^30
SPANS = {np.float64: [(-30, 20), (-20, 40), (-30, 60)], np.float32: [(-10, 10), (-12, 16), (-20, 25)]}


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2), (np.float64, 2), (np.float32, 3)])
@pytest.mark.parametrize("G", [300, 1024, 3000])
@pytest.mark.parametrize("span", [0, 1, 2])
def test_onchip_table_band_mode_zipf(R, dtype, K, G, span):
    R.set_kernel_variant(2)  # k_table
    try:
        rng = np.random.default_rng(G * 10 + span + K)
        n = (1 << 20) + 13
        lo, hi = SPANS[dtype][span]
        run(R, zipf_keys(rng, n, G), values(rng, n, dtype, lo, hi), G, K)
        assert R.last_path() == 0
    finally:
        R.set_kernel_variant(0)


@pytest.mark.parametrize("dtype,K,G", [(np.float64, 3, 1 << 16), (np.float32, 2, 1 << 17), (np.float32, 2, 1 << 20),
                                       (np.float64, 3, (1 << 20) - 7)])
def test_sweep_band_mode_zipf(R, dtype, K, G):
    # Zipf over G: a hot partition (summed in the scan pass) + cold partitions
    rng = np.random.default_rng(G + K)
    n = (1 << 21) + 5
    lo, hi = SPANS[dtype][1]
    run(R, zipf_keys(rng, n, G), values(rng, n, dtype, lo, hi), G, K)
    assert R.last_path() == 1


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2)])
def test_rows_above_and_below_the_band(R, dtype, K):
    # first rows of every block: tops 2 and 1 (band {1, 2}); later rows with
    # top 0 (below the band) and top 3 (above it) go to the slot table directly
    R.set_kernel_variant(2)
    try:
        rng = np.random.default_rng(5)
        G, n = 700, (1 << 20) + 1
        keys = zipf_keys(rng, n, G)
        big = (40, 60) if dtype == np.float64 else (15, 25)
        vals = values(rng, n, dtype, *big)
        sel = rng.random(n)
        tiny = (-40, -20) if dtype == np.float64 else (-15, -8)
        huge = (70, 100) if dtype == np.float64 else (31, 40)
        vals[sel < 0.3] = values(rng, int((sel < 0.3).sum()), dtype, *tiny)
        vals[sel > 0.999] = values(rng, int((sel > 0.999).sum()), dtype, *huge)
        run(R, keys, vals, G, K)
    finally:
        R.set_kernel_variant(0)


def test_band_then_uniform_switch(R):
    # uniform keys, values mostly at top 1 with a few top-0 groups early: the
    # first tile leaves groups untouched (band mode), all groups reach top 1
    # later (uniform mode), the last rows raise a few groups above the band
    R.set_kernel_variant(2)
    try:
        rng = np.random.default_rng(11)
        G, n = 2048, (1 << 21) + 3
        keys = rng.integers(0, G, n, dtype=np.int32)
        vals = values(rng, n, np.float64, -20, 20)
        vals[-50:] = values(rng, 50, np.float64, 30, 60)
        run(R, keys, vals, G, 3)
    finally:
        R.set_kernel_variant(0)


def test_hot_partition_band_with_heavy_groups(R):
    # config-3 shape at a small size: Zipf(1.1) over 2^20, binary32 normal * 2^e
    rng = np.random.default_rng(3)
    G, n = 1 << 20, (1 << 22) + 9
    keys = zipf_keys(rng, n, G)
    vals = (rng.standard_normal(n) * np.exp2(rng.integers(-10, 11, n))).astype(np.float32)
    run(R, keys, vals, G, 2)
    assert R.last_path() == 1


@pytest.mark.parametrize("bad", [-1, "G", "big"])
def test_hot_partition_pass_bad_keys(R, bad):
    # the hot pass classifies every row (hot / cold / bad key): a bad key
    # anywhere (in a hot block, late in the input) is EKEY, as in the oracle
    rng = np.random.default_rng(21)
    G, n = 1 << 20, (1 << 21) + 7
    keys = zipf_keys(rng, n, G)
    vals = (rng.standard_normal(n) * np.exp2(rng.integers(-10, 11, n))).astype(np.float32)
    keys[n - 5] = {-1: -1, "G": G, "big": 2 ** 31 - 1}[bad]
    assert O.groupby_sum(keys, vals, G, 2)[0] == O.EKEY
    with pytest.raises(R.ReproError) as ei:
        R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, 2)
    torch.cuda.synchronize()
    assert ei.value.status == O.EKEY


@pytest.mark.parametrize("offset", [1, 3])
def test_hot_partition_pass_unaligned(R, offset):
    # row arrays that are not 16-byte aligned take the scalar loads; the
    # compacted cold rows and the hot table must not care
    rng = np.random.default_rng(offset + 40)
    G, n = 1 << 20, (1 << 21) + 3
    keys = zipf_keys(rng, n, G)
    vals = (rng.standard_normal(n) * np.exp2(rng.integers(-10, 11, n))).astype(np.float32)
    kt = torch.zeros(n + offset, dtype=torch.int32, device="cuda")
    vt = torch.zeros(n + offset, dtype=torch.float32, device="cuda")
    kt[offset:] = torch.from_numpy(keys).cuda()
    vt[offset:] = torch.from_numpy(vals).cuda()
    out = R.groupby_sum(kt[offset:], vt[offset:], G, 2)
    torch.cuda.synchronize()
    rc, ref = O.groupby_sum(keys, vals, G, 2)
    assert rc == O.OK
    assert out.cpu().numpy().view(np.uint32).tobytes() == ref.view(np.uint32).tobytes()
    assert R.last_path() == 1


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float32, 2)])
@pytest.mark.parametrize("layout", ["sparse_parts", "one_big_many_tiny", "few_parts"])
def test_sweep_accumulate_schedule(R, dtype, K, layout):
    # the accumulate blocks' row ranges are cut on a cost scale (rows + one
    # table publish per partition): empty partitions, partitions of a few
    # rows next to one holding most rows, and cuts that snap to partition
    # starts all have to cover every row exactly once
    rng = np.random.default_rng(len(layout) * 10 + K)
    G = 1 << 20
    n = (1 << 21) + 13
    if layout == "sparse_parts":  # 5 partitions in use, the rest empty
        bases = np.array([0, 300000, 500000, 777777, G - 9])
        keys = bases[rng.integers(0, 5, n)] + rng.integers(0, 8, n)
    elif layout == "one_big_many_tiny":  # ~90% in one partition, 1-3 rows in many others
        keys = rng.integers(20000, 24000, n)
        tiny = rng.random(n) < 0.1
        keys[tiny] = rng.integers(0, G, int(tiny.sum()))
    else:  # uniform over 3 partitions' worth of groups, offset
        keys = rng.integers(9000, 9000 + 3 * 8192, n)
    keys = np.minimum(keys, G - 1).astype(np.int32)
    vals = (rng.standard_normal(n) * np.exp2(rng.integers(-12, 12, n))).astype(dtype)
    run(R, keys, vals, G, K)
