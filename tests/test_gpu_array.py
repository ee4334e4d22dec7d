"""GPU parity of the keyless single-array SUM and dot product (repro_sum /
repro_dot / repro_dot_async, f4 of SURVEY.md 8(f)) against the CPU oracle
(oracle.rsum / oracle.dot), bit for bit: sizes spanning several tiles with a
ragged tail, both formats and every fold, unaligned (register-load) inputs,
specials, cancellation and a full 2^27-element run."""
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


@pytest.fixture(params=[0, 3], ids=["register-kernel", "onchip-kernel"])
def variant(R, request):
    """0: the per-thread register kernel (k_array.cu, aligned arrays);
    3: the keyless on-chip GroupBy kernel with register loads."""
    R.set_kernel_variant(request.param)
    yield request.param
    R.set_kernel_variant(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def same(got, ref):
    return got.cpu().numpy().tobytes() == np.asarray([ref], dtype=got.cpu().numpy().dtype).tobytes()


def values(n, dtype, seed):
    _, v = synth.generate(1, n=n, seed=seed)  # +-(1+mant) 2^e, e in [-20, 20]
    return v.astype(dtype)


TILE64, TILE32 = 256 * 7, 256 * 15


@pytest.mark.parametrize("dtype,K", [(np.float64, 1), (np.float64, 2), (np.float64, 3), (np.float64, 4),
                                     (np.float32, 1), (np.float32, 2), (np.float32, 3), (np.float32, 4)])
@pytest.mark.parametrize("n", [1, 999, 5 * TILE32 + 17, (1 << 20) + 3])
def test_sum_parity(R, variant, dtype, K, n):
    x = values(n, dtype, 10 + n % 97)
    got = R.sum(dev(x), K)
    rc, ref = O.rsum(x, K)
    assert rc == O.OK
    assert same(got, ref)


@pytest.mark.parametrize("dtype,K", [(np.float64, 3), (np.float64, 2), (np.float32, 3), (np.float32, 1)])
@pytest.mark.parametrize("n", [7, 3 * TILE64 + 5, (1 << 20) + 1])
def test_dot_parity(R, variant, dtype, K, n):
    x, y = values(n, dtype, 1), values(n, dtype, 2)
    got = R.dot(dev(x), dev(y), K)
    rc, ref = O.dot(x, y, K)
    assert rc == O.OK
    assert same(got, ref)


@pytest.mark.parametrize("off", [1, 3])
def test_unaligned_inputs(R, off):
    """Views not 16-byte aligned take the register-load kernel."""
    n = 200001
    x = values(n + off, np.float64, 5)
    y = values(n + off, np.float64, 6)
    dx, dy = dev(x), dev(y)
    got_s = R.sum(dx[off:], 3)
    got_d = R.dot(dx[off:], dy[:n], 3)
    assert same(got_s, O.rsum(x[off:], 3)[1])
    assert same(got_d, O.dot(x[off:], y[:n], 3)[1])


def test_empty_and_zeros(R):
    z = R.sum(torch.zeros(0, dtype=torch.float64, device="cuda"), 3)
    assert z.cpu().numpy().view(np.uint64)[0] == 0
    z = R.sum(-torch.zeros(1000, dtype=torch.float64, device="cuda"), 3)
    assert z.cpu().numpy().view(np.uint64)[0] == 0


def test_cancellation_and_window(R, variant):
    for K, want in ((2, 0.0), (3, 1.0)):
        x = np.array([1.0, 2.0 ** 100] + [0.5] * 5000 + [-(2.0 ** 100)], dtype=np.float64)
        got = R.sum(dev(x), K)
        rc, ref = O.rsum(x, K)
        assert rc == O.OK and same(got, ref)
        if K == 3:
            assert ref == 2501.0
    x = np.full(1 << 20, 0.1)
    x[1::2] = -0.1
    assert R.sum(dev(x), 3).item() == 0.0


def test_specials_give_edom(R, variant):
    x = values(10000, np.float64, 3)
    x[1234] = np.nan
    x[5000] = 2.0 ** 1023  # k* = 27 > KMAX: ERANGE, lower precedence than EDOM
    with pytest.raises(R.ReproError) as e:
        R.sum(dev(x), 3)
    assert e.value.status == O.EDOM
    y = np.ones_like(x)
    x[5000] = 1.0
    x[1234] = np.inf
    y[1234] = 0.0  # inf * 0 = NaN
    with pytest.raises(R.ReproError) as e:
        R.dot(dev(x), dev(y), 3)
    assert e.value.status == O.EDOM
    x[1234] = 2.0 ** 1023
    with pytest.raises(R.ReproError) as e:
        R.sum(dev(x), 3)
    assert e.value.status == O.ERANGE
    assert O.rsum(x, 3)[0] == O.ERANGE


def test_level_shift_inside_a_thread(R, variant):
    """Large values late in the array (after a thread has deposited small
    ones) exercise the per-thread window raise and the block alignment."""
    n = 1 << 20
    x = values(n, np.float64, 11)
    x[n - 5000::997] = 2.0 ** 70 * 1.2345
    x[n // 2] = -(2.0 ** 90)
    for K in (1, 2, 3, 4):
        got = R.sum(dev(x), K)
        rc, ref = O.rsum(x, K)
        assert rc == O.OK and same(got, ref)


def test_async_form_and_dot_equals_sum_with_ones(R):
    n = 3 * TILE64 * 148 + 11
    x = values(n, np.float64, 8)
    dx = dev(x)
    ws = torch.empty(R.dot_workspace_bytes(3, R.F64) + 256, dtype=torch.uint8, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        R.dot_async(dx, None, 3, out, ws, status, stream=s)
    s.synchronize()
    assert status.item() == 0
    ref = O.rsum(x, 3)[1]
    assert same(out, ref)
    assert same(R.dot(dx, torch.ones_like(dx), 3), ref)
    # same bits as the keyed GroupBy with every key 0
    assert same(R.groupby_sum(torch.zeros(n, dtype=torch.int32, device="cuda"), dx, 1, 3), ref)


def test_full_size_sum(R):
    """2^27 elements (config 1's row count), one launch geometry as bench."""
    n = 1 << 27
    keys, x = synth.generate(1, n=n)
    got = R.sum(dev(x), 3)
    rc, ref = O.rsum(x, 3)
    assert rc == O.OK and same(got, ref)
    y = values(n, np.float64, 77)
    got = R.dot(dev(x), dev(y), 3)
    rc, ref = O.dot(x, y, 3)
    assert rc == O.OK and same(got, ref)


@pytest.mark.parametrize("ranks", [2, 3, 8])
def test_split_form_emulated_ranks(R, ranks):
    """The multi-GPU split form: each emulated rank deposits its shard into
    its own workspace; the slot tables are combined with the integer
    reductions dist.allreduce_table performs (OR / MAX / SUM) and read out --
    the same bits as one call over the whole array."""
    n = 1000003
    x = values(n, np.float64, 21)
    y = values(n, np.float64, 22)
    x[n // 3] = 2.0 ** 60  # one rank sees a higher window top than the others
    dx, dy = dev(x), dev(y)
    for yy, ref in ((None, O.rsum(x, 3)[1]), (dy, O.dot(x, y, 3)[1])):
        tables = []
        wss = []
        for r in range(ranks):
            a, b = n * r // ranks, n * (r + 1) // ranks
            ws = R.make_dot_workspace(3, R.F64)
            R.dot_deposit_async(dx[a:b], None if yy is None else yy[a:b], 3, ws)
            wss.append(ws)
            tables.append(R.dot_table_views(ws, 3, R.F64))
        f0, k0, s0 = tables[0]
        for f, k, s in tables[1:]:
            f0.copy_(f0 | f)
            k0.copy_(torch.maximum(k0, k))
            s0.add_(s)
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        R.dot_finish_async(3, R.F64, out, wss[0], status)
        torch.cuda.synchronize()
        assert status.item() == 0
        assert same(out, ref)
