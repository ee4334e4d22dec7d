"""The stream-ordered split form of the single-column GroupBy (SURVEY.md
8(e); repro_groupby_deposit_async / _finish_async / _window_limbs_async /
_finish_limbs_async) with emulated ranks on one GPU: each "rank" deposits its
shard into its own workspace; the collectives are replaced by the same
integer operations on the device (OR / MAX / SUM), so the result must equal
the oracle over all rows bit for bit, for any rank count, on both exchanges
(all-reduce of the slot table; reduce-scatter of the windowed limbs by group
range) and on both deposit paths (on-chip table, two-pass sweep)."""
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


def rows(G, n, dtype, seed):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-40, 41, n))).astype(dtype)
    vals[-3:] *= 2.0 ** 60 if dtype == np.float64 else 2.0 ** 20  # only the last shard sees the top windows
    return keys, vals


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("G,dtype,K", [(1024, np.float64, 3), (16, np.float32, 2), (50000, np.float64, 3),
                                       (70000, np.float32, 2),
                                       (8000, np.float64, 3), (16000, np.float32, 2)])  # (2-partition plans: replicated-read form)
def test_split_form_emulated_ranks(R, world, G, dtype, K):
    n = 300007
    keys, vals = rows(G, n, dtype, world + G)
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK
    dt = R.F64 if dtype == np.float64 else R.F32
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    nmax = -(-n // world)
    wss, views = [], []
    for r in range(world):
        a, b = r * n // world, (r + 1) * n // world
        ws = R.make_workspace(nmax, G, K, dt)
        R.groupby_deposit_async(torch.from_numpy(keys[a:b]).cuda(), torch.from_numpy(vals[a:b]).cuda(), G, K, ws)
        wss.append(ws)
        views.append(R.groupby_table_views(ws, nmax, G, K, dt))
    torch.cuda.synchronize()
    flags = torch.stack([v[0] for v in views]).max(0).values   # (no errors: OR == MAX)
    kglob = torch.stack([v[1] for v in views]).max(0).values
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    # exchange B: windowed limbs, summed, read out by group range
    limbs = []
    for r in range(world):
        lb = torch.empty(G * K * 2, dtype=torch.int64, device="cuda")
        R.groupby_window_limbs_async(nmax, G, K, dt, kglob, lb, wss[r])
        limbs.append(lb)
    summed = torch.stack(limbs).sum(0)
    per = -(-G // world)
    out2 = torch.empty(G, dtype=tdt, device="cuda")
    for r in range(world):
        g0, cnt = r * per, max(0, min(per, G - r * per))
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        R.groupby_finish_limbs_async(nmax, G, K, dt, g0, cnt, kglob[g0:g0 + cnt], summed[g0 * K * 2:(g0 + cnt) * K * 2],
                                     out2[g0:g0 + cnt], wss[r], st)
        torch.cuda.synchronize()
        assert st.item() == 0
    assert out2.cpu().numpy().tobytes() == ref.tobytes()
    # exchange A (after B: it overwrites rank 0's table with the sum)
    slots = torch.stack([v[2] for v in views]).sum(0)
    f0, k0, s0 = views[0]
    f0.copy_(flags)
    k0.copy_(kglob)
    s0.copy_(slots)
    out = torch.empty(G, dtype=tdt, device="cuda")
    R.groupby_finish_async(nmax, G, K, dt, out, wss[0], status)
    torch.cuda.synchronize()
    assert status.item() == 0
    assert out.cpu().numpy().tobytes() == ref.tobytes()


def test_split_form_errors_and_limits(R):
    G, K = 100, 3
    ws = R.make_workspace(1000, G, K, R.F64)
    keys = torch.zeros(1000, dtype=torch.int32, device="cuda")
    vals = torch.ones(1000, dtype=torch.float64, device="cuda")
    keys[7] = G  # EKEY reported by the finish
    R.groupby_deposit_async(keys, vals, G, K, ws)
    out = torch.empty(G, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    R.groupby_finish_async(1000, G, K, R.F64, out, ws, st)
    torch.cuda.synchronize()
    assert st.item() == R.EKEY
    # beyond the sweep's capacity the split form is not offered
    Gbig = R.sweep_max_groups(K, R.F64) + 1
    with pytest.raises(R.ReproError):
        R.groupby_table_views(torch.empty(1024, dtype=torch.uint8, device="cuda"), 10, Gbig, K, R.F64)


def test_acc_merge_with_itself_doubles(R):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 50, 20000, dtype=np.int32)
    vals = rng.standard_normal(20000)
    acc = R.Accumulator(50, 3, R.F64)
    acc.deposit(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    acc.merge(acc)
    rc, ref = O.groupby_sum(np.concatenate([keys, keys]), np.concatenate([vals, vals]), 50, 3)
    assert acc.finalize().cpu().numpy().tobytes() == ref.tobytes()
