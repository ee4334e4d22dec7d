"""GPU parity of the multi-column GroupBy (repro_groupby_sum_multi): several
SUMs + COUNT per key, fused into one on-chip pass for small group counts and
run column by column otherwise, against the CPU oracle bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from inputs import synth  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(R, keys, cols, G, K, proj, path=None):
    outs, counts = R.groupby_sum_multi(dev(keys), [dev(c) for c in cols], G, K, proj=proj)
    torch.cuda.synchronize()
    if path is not None:
        assert R.last_path() == path
    rc, ref, ref_counts = O.groupby_sum_multi(keys, cols, G, K, proj=proj)
    assert rc == O.OK
    for o, r in zip(outs, ref):
        assert o.cpu().numpy().tobytes() == r.tobytes()
    assert np.array_equal(counts.cpu().numpy(), ref_counts)


@pytest.fixture(params=[0, 1], ids=["lean-kernel", "onchip-kernel"])
def variant(R, request):
    """0: config-4 shapes with <= 4 groups take the per-thread register
    kernel (k_lean.cu); 1: force the shared-memory on-chip kernel."""
    R.set_kernel_variant(request.param)
    yield request.param
    R.set_kernel_variant(0)


@pytest.mark.parametrize("n", [1, 1000, 3 * 512 * 7 + 13, 1 << 20, (1 << 22) + 5])
def test_config4_shape_fused(R, variant, n):
    keys, (qty, price, disc, tax) = synth.generate(4, n=n)
    check(R, keys, [qty, price, disc, tax], 4, 3, 1, path=2)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_config4_shape_other_folds(R, variant, K):
    keys, cols = synth.generate(4, n=200003)
    check(R, keys, list(cols), 4, K, 1, path=2)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_config4_shape_fewer_groups(R, G):
    keys, cols = synth.generate(4, n=300001, n_groups=G)
    check(R, keys, list(cols), G, 3, 1, path=2)


@pytest.mark.parametrize("where", ["first", "middle", "last"])
@pytest.mark.parametrize("what", ["other_window", "zero", "tiny"])
def test_config4_lean_block_fallback(R, where, what):
    """A value off the block's lattice window (a larger or smaller k*, or a
    zero) sends that block through the generic code: same bits as the oracle."""
    n = 1 << 21
    keys, cols = synth.generate(4, n=n)
    cols = [c.copy() for c in cols]
    i = {"first": 0, "middle": n // 2 + 3, "last": n - 1}[where]
    if what == "other_window":
        cols[1][i] = 3.0e12  # price beyond 2^27: k* = 2
    elif what == "zero":
        cols[0][i] = 0.0     # qty 0: k* = 0 < 1
    else:
        cols[1][i] = 1.0e-9  # price below 2^-13: k* = 0
    check(R, keys, cols, 4, 3, 1, path=2)


@pytest.mark.parametrize("dtype,ncols,G", [(np.float64, 1, 4), (np.float64, 2, 3), (np.float64, 4, 1),
                                           (np.float32, 1, 2), (np.float32, 2, 4), (np.float32, 4, 4)])
def test_independent_columns_few_groups(R, variant, dtype, ncols, G):
    """Few groups: the lean kernel (variant 0) on single-window data, and on
    data spanning many windows (every block falls back)."""
    rng = np.random.default_rng(ncols * 100 + G)
    n = (1 << 20) + 7
    keys = rng.integers(0, G, n).astype(np.int32)
    one_window = [(rng.uniform(1, 2, n) * np.where(rng.random(n) < 0.5, -1, 1)).astype(dtype) for _ in range(ncols)]
    check(R, keys, one_window, G, 3 if dtype == np.float64 else 2, 0, path=2)
    spread = [(rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20, n)).astype(dtype) for _ in range(ncols)]
    check(R, keys, spread, G, 3 if dtype == np.float64 else 2, 0, path=2)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_moments_few_groups(R, variant, dtype):
    rng = np.random.default_rng(5)
    n = (1 << 20) + 3
    keys = rng.integers(0, 3, n).astype(np.int32)
    vals = (rng.uniform(1, 2, n) * 3.0).astype(dtype)
    got = R.groupby_moments(dev(keys), dev(vals), 3, 3)
    rc, ref = O.groupby_moments(keys, vals, 3, 3)
    assert rc == O.OK
    for k in ("sum", "avg", "var", "stddev", "count"):
        assert got[k].cpu().numpy().tobytes() == ref[k].tobytes(), k


def test_lean_kernel_is_the_one_that_runs(R):
    keys, cols = synth.generate(4, n=1 << 20)
    R.timing_enable(True)
    R.timing_collect()
    R.groupby_sum_multi(dev(keys), [dev(c) for c in cols], 4, 3, proj=1)
    torch.cuda.synchronize()
    names = R.timing_collect()
    R.timing_enable(False)
    assert "lean_multi" in names and "onchip_accumulate" not in names


def test_config4_lean_errors(R):
    keys, cols = synth.generate(4, n=1 << 20)
    cols = [c.copy() for c in cols]
    bad = cols[2].copy()
    bad[777777] = np.nan
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_multi(dev(keys), [dev(cols[0]), dev(cols[1]), dev(bad), dev(cols[3])], 4, 3, proj=1)
    assert e.value.status == R.EDOM
    k2 = keys.copy()
    k2[5] = 4
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_multi(dev(k2), [dev(c) for c in cols], 4, 3, proj=1)
    assert e.value.status == R.EKEY


@pytest.mark.parametrize("dtype,ncols,G", [(np.float64, 1, 7), (np.float64, 2, 100), (np.float64, 4, 200),
                                           (np.float32, 1, 33), (np.float32, 2, 5), (np.float32, 4, 50)])
def test_independent_columns_fused(R, dtype, ncols, G):
    rng = np.random.default_rng(ncols * 1000 + G)
    n = 300001
    keys = rng.integers(0, G, n).astype(np.int32)
    cols = [(rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20, n)).astype(dtype) for _ in range(ncols)]
    check(R, keys, cols, G, 3 if dtype == np.float64 else 2, 0, path=2)


@pytest.mark.parametrize("proj,ncols,G", [(1, 4, 300), (0, 3, 10), (0, 2, 5000)])
def test_column_by_column_fallback(R, proj, ncols, G):
    rng = np.random.default_rng(G)
    n = 250000
    if proj == 1:
        keys, cols = synth.generate(4, n=n, n_groups=G)
        cols = list(cols)
    else:
        keys = rng.integers(0, G, n).astype(np.int32)
        cols = [rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-40, 40, n) for _ in range(ncols)]
    check(R, keys, cols, G, 3, proj, path=3)


def test_unaligned_columns_take_register_loads(R):
    keys, cols = synth.generate(4, n=100001)
    # offset views: the columns are no longer 16-byte aligned (no TMA ring)
    kd = dev(np.concatenate([np.zeros(1, np.int32), keys]))[1:]
    cd = [dev(np.concatenate([[0.0], c]))[1:] for c in cols]
    outs, counts = R.groupby_sum_multi(kd, cd, 4, 3, proj=1)
    rc, ref, rc_counts = O.groupby_sum_multi(keys, list(cols), 4, 3, proj=1)
    for o, r in zip(outs, ref):
        assert o.cpu().numpy().tobytes() == r.tobytes()
    assert np.array_equal(counts.cpu().numpy(), rc_counts)


def test_multi_level_shifts_and_order_invariance(R):
    rng = np.random.default_rng(3)
    n = 400000
    keys = rng.integers(0, 6, n).astype(np.int32)
    cols = [rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-200, 200, n) for _ in range(2)]
    check(R, keys, cols, 6, 3, 0, path=2)
    perm = rng.permutation(n)
    a, _ = R.groupby_sum_multi(dev(keys), [dev(c) for c in cols], 6, 3)
    b, _ = R.groupby_sum_multi(dev(keys[perm]), [dev(c[perm]) for c in cols], 6, 3)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_multi_errors(R):
    keys = np.zeros(5000, np.int32)
    good = np.ones(5000)
    bad = good.copy()
    bad[1234] = np.nan
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_multi(dev(keys), [dev(good), dev(bad)], 2, 3)
    assert e.value.status == R.EDOM
    keys[77] = 9
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_multi(dev(keys), [dev(good), dev(bad)], 2, 3)
    assert e.value.status == R.EKEY
    with pytest.raises(R.ReproError) as e:  # projection needs 4 binary64 columns
        R.groupby_sum_multi(dev(keys), [dev(good)] * 3, 2, 3, proj=1)
    assert e.value.status == R.EINVAL


def test_multi_async_matches_blocking(R):
    keys, cols = synth.generate(4, n=123457)
    kd, cd = dev(keys), [dev(c) for c in cols]
    ws = R.make_multi_workspace(keys.size, 4, 4, 1, 3, R.F64)
    st = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    outs = [torch.empty(4, dtype=torch.float64, device="cuda") for _ in range(4)]
    counts = torch.empty(4, dtype=torch.int64, device="cuda")
    R.groupby_sum_multi_async(kd, cd, 4, 3, 1, outs, counts, ws, st)
    torch.cuda.synchronize()
    assert st.item() == 0
    ref, rc = R.groupby_sum_multi(kd, cd, 4, 3, proj=1)
    for x, y in zip(outs, ref):
        assert torch.equal(x, y)
    assert torch.equal(counts, rc)


def test_split_form_with_emulated_ranks(R):
    # the multi-GPU split form on one GPU: two "ranks" deposit their halves into
    # their own workspaces; their slot tables are combined the way
    # dist.allreduce_table combines them (OR / MAX / SUM), then read out
    keys, cols = synth.generate(4, n=300007)
    kd, cd = dev(keys), [dev(c) for c in cols]
    n, G, K = keys.size, 4, 3
    h = n // 2
    wss = [R.make_multi_workspace(n, G, 4, 1, K, R.F64) for _ in range(2)]
    for w, (a, b) in zip(wss, ((0, h), (h, n))):
        R.groupby_multi_deposit_async(kd[a:b], [c[a:b] for c in cd], G, K, 1, w)
    t0 = R.multi_table_views(wss[0], n, G, 4, 1, K, R.F64)
    t1 = R.multi_table_views(wss[1], n, G, 4, 1, K, R.F64)
    t0[0].copy_(t0[0] | t1[0])
    torch.maximum(t0[1], t1[1], out=t0[1])
    t0[2].add_(t1[2])
    outs = [torch.empty(G, dtype=torch.float64, device="cuda") for _ in range(4)]
    counts = torch.empty(G, dtype=torch.int64, device="cuda")
    st = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    R.groupby_multi_finish_async(n, G, 4, 1, K, R.F64, outs, counts, wss[0], st)
    torch.cuda.synchronize()
    assert st.item() == 0
    ref, rc = R.groupby_sum_multi(kd, cd, G, K, proj=1)
    for x, y in zip(outs, ref):
        assert torch.equal(x, y)
    assert torch.equal(counts, rc)


@pytest.mark.parametrize("dtype,G,n", [(np.float64, 10, 200003), (np.float32, 7, 100001), (np.float64, 700, 50001)])
def test_moments_match_oracle(R, dtype, G, n):
    rng = np.random.default_rng(G + n)
    keys = rng.integers(0, G, n).astype(np.int32)
    x = (rng.standard_normal(n) * 2.0 ** rng.integers(-10, 10, n)).astype(dtype)
    res = R.groupby_moments(dev(keys), dev(x), G, 3 if dtype == np.float64 else 2)
    rc, ref = O.groupby_moments(keys, x, G, 3 if dtype == np.float64 else 2)
    assert rc == O.OK
    for k in ("sum", "avg", "var", "stddev", "count"):
        assert res[k].cpu().numpy().tobytes() == ref[k].tobytes(), k
