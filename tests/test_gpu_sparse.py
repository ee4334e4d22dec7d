"""GPU parity of the arbitrary-key GroupBy (repro_groupby_sum_sparse, SURVEY.md
8(f) f1): hash-mapped dense ids + the dense reproducible path, against the
oracle (np.unique + O5), bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("dtype,distinct,n,K", [(np.float64, 37, 200003, 3), (np.float32, 1000, 300001, 2),
                                                 (np.float64, 20000, 400000, 3), (np.float64, 1, 5000, 2)])
def test_sparse_matches_oracle(R, dtype, distinct, n, K):
    rng = np.random.default_rng(distinct + n)
    pool = np.unique(rng.integers(-(1 << 62), 1 << 62, distinct * 2))[:distinct]
    keys = pool[rng.integers(0, pool.size, n)]
    vals = (rng.standard_normal(n) * 2.0 ** rng.integers(-30, 30, n)).astype(dtype)
    uk, out = R.groupby_sum_sparse(dev(keys), dev(vals), max_groups=2 * distinct, fold=K)
    rc, ruk, rout = O.groupby_sum_sparse(keys, vals, K)
    assert rc == O.OK
    assert np.array_equal(uk.cpu().numpy(), ruk)
    assert out.cpu().numpy().tobytes() == rout.tobytes()
    perm = rng.permutation(n)
    uk2, out2 = R.groupby_sum_sparse(dev(keys[perm]), dev(vals[perm]), max_groups=2 * distinct, fold=K)
    assert torch.equal(uk, uk2) and torch.equal(out, out2)


@pytest.mark.parametrize("lo,distinct", [(-2500, 5000), (1 << 40, 70000), (-(1 << 62), 3)])
def test_sparse_dense_key_runs(R, lo, distinct):
    # consecutive keys share their high digits: every radix pass but the low
    # ones sees long runs of equal digits (stability decides the order)
    rng = np.random.default_rng(distinct)
    n = 8 * distinct + 11
    keys = (lo + rng.integers(0, distinct, n)).astype(np.int64)
    keys[:distinct] = lo + np.arange(distinct)  # every key present
    vals = (rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20, n)).astype(np.float64)
    uk, out = R.groupby_sum_sparse(dev(keys), dev(vals), max_groups=distinct + 7, fold=3)
    rc, ruk, rout = O.groupby_sum_sparse(keys, vals, 3)
    assert rc == O.OK
    assert np.array_equal(uk.cpu().numpy(), ruk)
    assert np.array_equal(ruk, lo + np.arange(distinct))
    assert out.cpu().numpy().tobytes() == rout.tobytes()


def test_sparse_capacity_and_errors(R):
    keys = np.arange(5000, dtype=np.int64) * 7919
    vals = np.ones(5000)
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_sparse(dev(keys), dev(vals), max_groups=100)
    assert e.value.status == R.ENOMEM
    keys[17] = np.iinfo(np.int64).min
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_sparse(dev(keys), dev(vals), max_groups=8000)
    assert e.value.status == R.EKEY
    uk, out = R.groupby_sum_sparse(dev(np.zeros(0, np.int64)), dev(np.zeros(0)), max_groups=10)
    assert uk.numel() == 0 and out.numel() == 0


@pytest.mark.parametrize("dtype,distinct,n,K", [(np.float64, 500, 300007, 3), (np.float32, 30000, 400001, 2)])
def test_sparse_int32_keys_match_oracle(R, dtype, distinct, n, K):
    # every int32 value is a valid key (INT32_MIN included); out_keys int64
    rng = np.random.default_rng(distinct)
    pool = np.unique(np.concatenate([[np.iinfo(np.int32).min, np.iinfo(np.int32).max, 0, -1],
                                     rng.integers(-(1 << 31), (1 << 31) - 1, distinct * 2)]))[:distinct]
    keys = pool[rng.integers(0, pool.size, n)].astype(np.int32)
    vals = (rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20, n)).astype(dtype)
    uk, out = R.groupby_sum_sparse(dev(keys), dev(vals), max_groups=2 * distinct, fold=K)
    rc, ruk, rout = O.groupby_sum_sparse(keys.astype(np.int64), vals, K)
    assert rc == O.OK
    assert uk.dtype == torch.int64 and np.array_equal(uk.cpu().numpy(), ruk)
    assert out.cpu().numpy().tobytes() == rout.tobytes()
    # the same multiset as int64 keys gives the same bits
    uk64, out64 = R.groupby_sum_sparse(dev(keys.astype(np.int64)), dev(vals), max_groups=2 * distinct, fold=K)
    assert torch.equal(uk, uk64) and torch.equal(out, out64)
