"""GPU parity on the edge cases of the accumulator's domain, for every code
path and both formats (VERDICT r1 "parity gaps"):

  * window-top thresholds 2^(W k + W - 1 - m) and the values just below them
    (Alg. 1 line 3), up to the ERANGE limit (reading A-9);
  * subnormals and signed zeros (reading A-11);
  * half-unit ties (d + 1/2) u_l at every level, both signs (reading A-1);
  * the binary32 carry-count limit |C| >= 2^24 (reading A-8);
  * a pending dynamic fold together with a bad row (the fast-path
    check must run whatever the fold bit says).

Paths: the lean per-warp kernel (<= 16 groups), the on-chip kernel (TMA ring
and register loads), the partitioned path (forced) and the keyless k_rsum.
Expected values come only from the oracle (and closed forms for the carry
limit).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402  (test infrastructure)
import edge_values as EV  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


PATHS = ["auto", "onchip_tma", "onchip_reg", "partitioned"]


@pytest.fixture(params=PATHS)
def path(R, request):
    p = request.param
    if p == "onchip_tma":
        R.set_kernel_variant(1)
    elif p == "onchip_reg":
        R.set_kernel_variant(3)
    elif p == "partitioned":
        R.set_path_override(1)
    yield p
    R.set_kernel_variant(0)
    R.set_path_override(-1)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(R, keys, vals, G, K):
    out = torch.empty(G, dtype=torch.float64 if vals.dtype == np.float64 else torch.float32, device="cuda")
    try:
        R.groupby_sum(dev(keys), dev(vals), G, K, out=out)
        torch.cuda.synchronize()
        return 0, out.cpu().numpy()
    except R.ReproError as e:
        return e.status, None


def check(R, keys, vals, G, K):
    rc, ref = O.groupby_sum(keys, vals, G, K)
    st, got = run(R, keys, vals, G, K)
    assert st == rc, (st, rc)
    if rc == 0:
        bits = np.uint64 if vals.dtype == np.float64 else np.uint32
        bad = np.nonzero(got.view(bits) != ref.view(bits))[0]
        assert bad.size == 0, f"{bad.size} groups differ, first {bad[:4]}: {got[bad[:4]]} vs {ref[bad[:4]]}"
    return rc


@pytest.mark.parametrize("bits,K", [(64, 3), (64, 2), (32, 2), (32, 3)])
@pytest.mark.parametrize("G", [8, 300])
def test_edge_rows_match_oracle(R, path, bits, K, G):
    rng = np.random.default_rng(7000 + bits + 10 * K + G)
    keys, vals = EV.edge_rows(rng, bits, K, G, 60001)
    assert check(R, keys, vals, G, K) == 0


@pytest.mark.parametrize("bits,K", [(64, 3), (32, 2)])
def test_edge_single_window_blocks(R, path, bits, K):
    # every value of every group at window 1 (ties, thresholds below it,
    # subnormals, zeros): the lean kernel's one-window blocks and the on-chip
    # fast path take these without falling back
    rng = np.random.default_rng(8000 + bits + K)
    pool = np.array(EV.ties(bits, K, 1) + [EV.anchor(bits, 1)] + EV.subnormals(bits) +
                    [v for v in EV.thresholds(bits) if abs(v) < EV.threshold(1, bits)], dtype=EV.np_type(bits))
    n, G = 200003, 12
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = pool[rng.integers(0, pool.size, n)]
    vals[rng.integers(0, n, 64)] = EV.anchor(bits, 1)
    assert check(R, keys, vals, G, K) == 0


@pytest.mark.parametrize("bits", [64, 32])
def test_erange_limit_every_path(R, path, bits):
    t = EV.np_type(bits)
    lim = EV.erange_limit(bits)
    rng = np.random.default_rng(9)
    n, G = 50000, 40
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = rng.standard_normal(n).astype(t)
    K = 3 if bits == 64 else 2
    for where in (17, n // 2, n - 5):
        v = vals.copy()
        v[where] = EV.below(lim, bits)          # largest value with a finite extractor: OK
        v[(where + 101) % n] = -EV.below(lim, bits)
        assert check(R, keys, v, G, K) == 0
        v[where] = lim                           # the limit itself: ERANGE
        assert check(R, keys, v, G, K) == O.ERANGE
        v[where] = -lim
        assert check(R, keys, v, G, K) == O.ERANGE


@pytest.mark.parametrize("bits,dtype", [(64, np.float64), (32, np.float32)])
def test_subnormals_and_zeros_every_path(R, path, bits, dtype):
    sub = np.array(EV.subnormals(bits), dtype)
    rng = np.random.default_rng(11)
    n, G = 40000, 20
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = sub[rng.integers(0, sub.size, n)]
    rc, ref = O.groupby_sum(keys, vals, G, 2)
    st, got = run(R, keys, vals, G, 2)
    assert rc == st == 0
    assert got.tobytes() == ref.tobytes() == np.zeros(G, dtype).tobytes()  # +0.0 everywhere
    # mixed with normal values: subnormals contribute nothing at f = 0
    vals2 = vals.copy()
    vals2[::3] = rng.standard_normal(vals2[::3].size).astype(dtype)
    assert check(R, keys, vals2, G, 3) == 0


@pytest.mark.parametrize("bits", [64, 32])
def test_keyless_sum_edges(R, bits):
    # k_rsum (f4): the same edge values through the single-array SUM
    rng = np.random.default_rng(12)
    t = EV.np_type(bits)
    K = 3 if bits == 64 else 2
    for kt in (0, 1, 2):
        pool = np.array(EV.edge_pool(bits, K, kt), dtype=t)
        for n in (1, 37, 100003):
            x = pool[rng.integers(0, pool.size, n)]
            rc, ref = O.rsum(x, K)
            try:
                got = R.sum(dev(x), K).cpu().numpy()[0]
                st = 0
            except R.ReproError as e:
                st = e.status
            assert st == rc
            if rc == 0:
                assert np.array([got]).tobytes() == np.array([ref], dtype=t).tobytes(), (kt, n, got, ref)
        x = pool[rng.integers(0, pool.size, 5000)].copy()
        x[4000] = EV.erange_limit(bits)
        with pytest.raises(R.ReproError) as e:
            R.sum(dev(x), K)
        assert e.value.status == O.ERANGE


# ---------------------------------------------------------------------------
# binary32 carry-count limit (reading A-8)
# ---------------------------------------------------------------------------

def _f32_state(cs):
    # canonical k = 0 states with D = 0 and C_1 = c (SPEC.md:277 layout:
    # S[0..K) then C[0..K) per group)
    st = np.zeros((len(cs), 4), np.float32)
    st[:, 0], st[:, 1] = 1.5, 1.5 * 2.0 ** -18
    st[:, 2] = cs
    return dev(st.reshape(-1))


def test_f32_carry_limit_imported_state(R):
    # |C| < 2^24 reads out C / 4; a merge that reaches |C| = 2^24 is ERANGE at
    # read-out (reading A-8); importing |C| >= 2^24 is EINVAL (no canonical
    # binary32 state the accumulator can export holds it)
    cs = (2.0 ** 24 - 1, -(2.0 ** 24 - 1), 12345.0)
    acc = R.Accumulator(3, 2, R.F32)
    acc.import_(_f32_state(cs))
    got = acc.finalize().cpu().numpy()
    p = O.params(O.F32, 2)
    ref = [O.finalize(p, O.State([1.5, 1.5 * 2.0 ** -18], [float(c), 0.0])) for c in cs]
    assert got.tolist() == ref == [float(np.float32(c / 4)) for c in cs]
    with pytest.raises(R.ReproError) as e:
        acc.import_(_f32_state((2.0 ** 24, 0.0, 0.0)))
    assert e.value.status == O.EINVAL
    a, b = R.Accumulator(3, 2, R.F32), R.Accumulator(3, 2, R.F32)
    a.import_(_f32_state((2.0 ** 23, -(2.0 ** 23), 2.0 ** 23 - 1)))
    b.import_(_f32_state((2.0 ** 23, -(2.0 ** 23), 2.0 ** 23)))
    a.merge(b)  # C = 2^24, -2^24, 2^24 - 1
    with pytest.raises(R.ReproError) as e:
        a.finalize()
    assert e.value.status == O.ERANGE
    # the oracle's merge of the same states agrees
    sa, sb = O.State([1.5, 1.5 * 2.0 ** -18], [2.0 ** 23, 0.0]), O.State([1.5, 1.5 * 2.0 ** -18], [2.0 ** 23, 0.0])
    assert O.merge(p, sa, sb) == O.OK
    with pytest.raises(ValueError, match=str(O.ERANGE)):
        O.finalize(p, sa)


@pytest.mark.parametrize("path_kind", ["auto", "onchip", "partitioned"])
def test_f32_carry_limit_by_rows(R, path_kind):
    # b = the largest binary32 below 2^-6 carries C_1 = n / 16 in one group:
    # n = 2^28 rows reach C = 2^24 (ERANGE); n = 2^28 - 16 reads out 2^22 - 1/2
    b = np.float32(EV.below(2.0 ** -6, 32))
    n = 1 << 28
    vals = torch.full((n,), float(b), dtype=torch.float32, device="cuda")
    keys = torch.zeros(n, dtype=torch.int32, device="cuda")
    G = 1 if path_kind == "auto" else 40  # 40 groups (others empty) leaves the lean kernel
    if path_kind == "onchip":
        R.set_kernel_variant(1)
    elif path_kind == "partitioned":
        R.set_path_override(1)
    try:
        with pytest.raises(R.ReproError) as e:
            R.groupby_sum(keys, vals, G, 2)
        assert e.value.status == O.ERANGE
        out = R.groupby_sum(keys[: n - 16], vals[: n - 16], G, 2).cpu().numpy()
        assert float(out[0]) == 2.0 ** 22 - 0.5 and not out[1:].any()
    finally:
        R.set_kernel_variant(0)
        R.set_path_override(-1)
    # and the oracle on the same rows (host copies)
    hk, hv = np.zeros(n - 16, np.int32), np.full(n - 16, b, np.float32)
    rc, ref = O.groupby_sum(hk, hv, 1, 2)
    assert rc == 0 and float(ref[0]) == 2.0 ** 22 - 0.5


# ---------------------------------------------------------------------------
# dynamic fold + bad rows: a pending fold must not skip the
# fast path's row checks
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("G", [33, 200, 1024])
@pytest.mark.parametrize("bad", ["key", "nan", "big"])
def test_fold_pending_with_bad_row(R, G, bad):
    R.set_kernel_variant(1)
    try:
        rng = np.random.default_rng(G)
        n = 1 << 22
        # three groups of the G-group table hold all rows (thousands per group
        # per block); values just below the window top, all of one sign, climb
        # the counters to 2^30 and trigger the dynamic fold again and again
        keys = rng.choice(np.array([0, 1, G - 1], np.int32), n)
        vals = np.full(n, EV.below(EV.threshold(1, 64), 64), np.float64) * rng.uniform(0.9, 1.0, n)
        idx = rng.integers(n // 2, n, 24)
        if bad == "key":
            keys[idx] = G + 3
            want = O.EKEY
        elif bad == "nan":
            vals[idx] = np.nan
            want = O.EDOM
        else:
            vals[idx] = 2.0 ** 60  # window raise late in a block: no error, parity
            want = 0
        assert check(R, keys, vals, G, 3) == want
    finally:
        R.set_kernel_variant(0)
