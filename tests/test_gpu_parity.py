"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, bit
for bit (the type is associative, so the north star's bar is bit-exact).

Sizes span several tiles (1792 rows per tile for binary64, 3840 for binary32,
one tile per 256 x R rows) and ragged tails; the full BASELINE sizes are
covered in test_gpu_full_size.py.  The `variant` fixture runs the on-chip
cases under k_table, the TMA-fed kernel and the register-load kernel (unaligned inputs take that path too).
"""
import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402  (test infrastructure)
from inputs import synth  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


@pytest.fixture(params=[0, 1, 2, 3], ids=["auto", "atomic", "table", "regload"])
def variant(R, request):
    """Run a test under each on-chip kernel (auto: the lean per-warp kernel for
    <= 16 groups, else k_table / TMA-fed per-row atomics / k_table / per-row
    atomics with register loads)."""
    R.set_kernel_variant(request.param)
    yield request.param
    R.set_kernel_variant(0)


def dtype_code(dtype):
    return 1 if dtype == np.float64 else 0


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_groupby(R, keys, vals, G, K):
    out = R.groupby_sum(dev(keys), dev(vals), G, K)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def oracle_groupby(keys, vals, G, K):
    rc, out = O.groupby_sum(keys, vals, G, K)
    assert rc == O.OK, rc
    return out


def mixed_values(rng, n, dtype, spread):
    e = rng.integers(-spread, spread + 1, n)
    v = rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1.0, 1.0], n)
    v[rng.random(n) < 0.02] = 0.0
    return v.astype(dtype)


def assert_bits_equal(a, b):
    assert a.dtype == b.dtype
    ia = a.view(np.uint64 if a.dtype == np.float64 else np.uint32)
    ib = b.view(np.uint64 if b.dtype == np.float64 else np.uint32)
    bad = np.nonzero(ia != ib)[0]
    assert bad.size == 0, f"{bad.size} groups differ, first {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"


# ---------------------------------------------------------------- config 0

def test_config0_matches_oracle(R, variant):
    keys, vals = synth.generate(0)
    assert_bits_equal(gpu_groupby(R, keys, vals, 16, 3), oracle_groupby(keys, vals, 16, 3))


def test_config0_state_export_matches_oracle(R):
    keys, vals = synth.generate(0)
    acc = R.Accumulator(16, 3, R.F64)
    acc.deposit(dev(keys), dev(vals))
    st = acc.export().cpu().numpy().reshape(16, 6)
    rc, out, ost = O.groupby_sum(keys, vals, 16, 3, with_state=True)
    assert rc == O.OK
    assert st.view(np.uint64).tolist() == ost.view(np.uint64).tolist()


# --------------------------------------------------- three-row example (P-1)

@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_three_row_example_all_permutations(R, variant, K):
    base = [2.5e-16, 0.999999999999999, 2.5e-16]
    ref = None
    for perm in itertools.permutations(base):
        vals = np.array(list(perm) * 5000, dtype=np.float64)  # 15000 rows, several tiles
        keys = np.zeros(vals.size, dtype=np.int32)
        got = gpu_groupby(R, keys, vals, 1, K)
        ref = oracle_groupby(keys, vals, 1, K) if ref is None else ref
        assert_bits_equal(got, ref)


# -------------------------------------------------- randomized shapes / dtypes

CASES = [
    # (dtype, K, G, n, spread)
    (np.float64, 3, 1024, 3 * 3072 * 7 + 17, 20),
    (np.float64, 1, 16, 100003, 60),
    (np.float64, 2, 333, 250001, 90),
    (np.float64, 4, 77, 50000, 200),
    (np.float64, 3, 1, 40000, 30),
    (np.float64, 3, 2, 77777, 300),       # per-lane counter copies, level shifts
    (np.float64, 3, 32, 123457, 120),     # largest G with per-lane copies
    (np.float64, 3, 33, 123457, 120),     # smallest G without
    (np.float32, 2, 32, 98765, 40),
    (np.float32, 2, 1024, 4096 * 9 + 5, 10),
    (np.float32, 1, 5, 70001, 40),
    (np.float32, 3, 2000, 300007, 30),
    (np.float32, 4, 64, 65536, 60),
]


@pytest.mark.parametrize("dtype,K,G,n,spread", CASES)
def test_random_matches_oracle(R, variant, dtype, K, G, n, spread):
    rng = np.random.default_rng(n + G + K)
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = mixed_values(rng, n, dtype, spread)
    assert_bits_equal(gpu_groupby(R, keys, vals, G, K), oracle_groupby(keys, vals, G, K))


def test_level_shift_late_in_block(R, variant):
    # small values first, then a huge value late in the same block: the tile-phase
    # demotion must shift the already accumulated level sums
    n = 200000
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 8, n, dtype=np.int32)
    vals = rng.uniform(-1e-6, 1e-6, n)
    vals[-3] = 2.0 ** 100
    vals[n // 2] = -(2.0 ** 60)
    vals[n // 3] = 2.0 ** 45
    assert_bits_equal(gpu_groupby(R, keys, vals, 8, 3), oracle_groupby(keys, vals, 8, 3))


def test_hot_group_skew(R, variant):
    # Zipf-like skew: most rows in one group (warp-aggregated path)
    keys, vals = synth.generate_chunked(3, 1 << 18, 1 << 10)
    assert_bits_equal(gpu_groupby(R, keys, vals, 1 << 10, 2), oracle_groupby(keys, vals, 1 << 10, 2))


def test_row_permutation_invariance_on_gpu(R, variant):
    keys, vals = synth.generate_chunked(1, 1 << 20, 1024)
    ref = gpu_groupby(R, keys, vals, 1024, 3)
    rng = np.random.default_rng(9)
    for _ in range(2):
        p = rng.permutation(keys.size)
        assert_bits_equal(gpu_groupby(R, keys[p], vals[p], 1024, 3), ref)
    assert_bits_equal(ref, oracle_groupby(keys, vals, 1024, 3))


# ------------------------------------------------------------------ edge cases

def test_empty_input(R):
    out = gpu_groupby(R, np.zeros(0, np.int32), np.zeros(0), 7, 3)
    assert out.tobytes() == np.zeros(7).tobytes()


def test_empty_groups_and_cancellation_are_positive_zero(R, variant):
    keys = np.array([1, 1, 3, 3, 3], np.int32)
    vals = np.array([2.5, -2.5, 1e290, -1e290, 0.0])
    out = gpu_groupby(R, keys, vals, 5, 3)
    assert out.tobytes() == np.zeros(5).tobytes()


def test_single_row_round_trip(R, variant):
    rng = np.random.default_rng(12)
    v = rng.uniform(1, 2, 1000) * np.exp2(rng.integers(-80, 900, 1000))
    keys = np.arange(1000, dtype=np.int32)
    out = gpu_groupby(R, keys, v, 1000, 3)
    assert_bits_equal(out, v)


def test_max_onchip_groups(R, variant):
    for dtype, K in ((np.float64, 3), (np.float32, 2)):
        G = R.onchip_max_groups(K, R.F64 if dtype == np.float64 else R.F32)
        assert G >= 1024
        rng = np.random.default_rng(G)
        n = 5 * G + 11
        keys = rng.integers(0, G, n, dtype=np.int32)
        vals = mixed_values(rng, n, dtype, 20)
        assert_bits_equal(gpu_groupby(R, keys, vals, G, K), oracle_groupby(keys, vals, G, K))
        assert R.last_path() == 0


@pytest.mark.parametrize("bad,code", [("key", -2), ("neg", -2), ("nan", -3), ("inf", -3), ("big", -4)])
def test_device_errors(R, bad, code):
    keys = np.zeros(10000, np.int32)
    vals = np.ones(10000)
    if bad == "key":
        keys[5000] = 9
    elif bad == "neg":
        keys[77] = -1
    elif bad == "nan":
        vals[9999] = np.nan
    elif bad == "inf":
        vals[0] = -np.inf
    else:
        vals[1234] = 2.0 ** 990
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 4, 3)
    assert ei.value.status == code
    assert O.groupby_sum(keys, vals, 4, 3)[0] == code


def test_error_precedence(R):
    keys = np.zeros(1000, np.int32)
    vals = np.ones(1000)
    vals[10] = np.nan
    vals[20] = 2.0 ** 1000
    keys[900] = 50
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 4, 3)
    assert ei.value.status == R.EKEY
    keys[900] = 0
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 4, 3)
    assert ei.value.status == R.EDOM


def test_fp32_range_error(R):
    keys = np.zeros(3, np.int32)
    vals = np.array([1.0, 2.0 ** 120, 1.0], np.float32)
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 1, 2)
    assert ei.value.status == R.ERANGE


def test_bad_arguments(R):
    k = dev(np.zeros(4, np.int32))
    v = dev(np.ones(4))
    with pytest.raises(R.ReproError):
        R.groupby_sum(k, v, 0, 3)
    with pytest.raises(R.ReproError):
        R.groupby_sum(k, v, 4, 5)


# ------------------------------------------------------------ accumulator API

def test_acc_chunked_deposits_and_merge_equal_one_shot(R):
    keys, vals = synth.generate_chunked(1, 1 << 20, 1024)
    ref = oracle_groupby(keys, vals, 1024, 3)
    a = R.Accumulator(1024, 3, R.F64)
    cuts = [0, 1, 4097, 300000, 777777, keys.size]
    for c0, c1 in zip(cuts[:-1], cuts[1:]):
        a.deposit(dev(keys[c0:c1]), dev(vals[c0:c1]))
    assert_bits_equal(a.finalize().cpu().numpy(), ref)
    b1, b2 = R.Accumulator(1024, 3, R.F64), R.Accumulator(1024, 3, R.F64)
    b1.deposit(dev(keys[::2]), dev(vals[::2]))
    b2.deposit(dev(keys[1::2]), dev(vals[1::2]))
    b2.merge(b1)
    assert_bits_equal(b2.finalize().cpu().numpy(), ref)
    assert torch.equal(b2.export(), a.export())


def test_acc_export_import_round_trip(R):
    rng = np.random.default_rng(3)
    for dtype, dt, K in ((np.float64, R.F64, 3), (np.float32, R.F32, 2)):
        keys = rng.integers(0, 50, 20000, dtype=np.int32)
        vals = mixed_values(rng, 20000, dtype, 30)
        a = R.Accumulator(50, K, dt)
        a.deposit(dev(keys), dev(vals))
        st = a.export()
        b = R.Accumulator(50, K, dt).import_(st)
        assert torch.equal(b.finalize(), a.finalize())
        assert torch.equal(b.export(), st)
        rc, out, ost = O.groupby_sum(keys, vals, 50, K, with_state=True)
        assert st.cpu().numpy().astype(np.float64).reshape(50, 2 * K).tobytes() == ost.tobytes()
        bad = st.clone()
        bad[0] = 1.0  # S^(1) = 1.0 is not a canonical running sum
        with pytest.raises(R.ReproError):
            R.Accumulator(50, K, dt).import_(bad)


def test_window_exchange_emulates_ranks(R):
    # two "ranks" on one GPU: all-reduce MAX on k and SUM on limbs done with torch
    keys, vals = synth.generate_chunked(1, 1 << 19, 1024)
    vals = vals.copy()
    vals[:1000] *= 2.0 ** 70  # rank 0 needs a higher window for some groups
    ref = oracle_groupby(keys, vals, 1024, 3)
    accs = []
    for r in range(2):
        a = R.Accumulator(1024, 3, R.F64)
        a.deposit(dev(keys[r::2]), dev(vals[r::2]))
        accs.append(a)
    kg = torch.maximum(accs[0].top_levels(), accs[1].top_levels())
    limbs = accs[0].window_export(kg) + accs[1].window_export(kg)
    accs[1].window_import(kg, limbs)
    assert_bits_equal(accs[1].finalize().cpu().numpy(), ref)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_reduce_scatter_exchange_emulates_ranks(R, world):
    """dist.reduce_scatter_finalize's steps on one GPU: each emulated rank
    imports only its contiguous group range (window_import range form) and
    finalises it; the concatenated ranges equal the oracle."""
    G = 1000  # not a multiple of world
    keys, vals = synth.generate_chunked(1, 1 << 19, G)
    vals = vals.copy()
    vals[:1000] *= 2.0 ** 70
    ref = oracle_groupby(keys, vals, G, 3)
    accs = []
    for r in range(world):
        a = R.Accumulator(G, 3, R.F64)
        a.deposit(dev(keys[r::world]), dev(vals[r::world]))
        accs.append(a)
    kg = accs[0].top_levels()
    for a in accs[1:]:
        kg = torch.maximum(kg, a.top_levels())
    limbs = sum(a.window_export(kg) for a in accs)
    per = -(-G // world)
    parts = []
    for r, a in enumerate(accs):
        g0, cnt = r * per, max(0, min(per, G - r * per))
        if cnt:
            a.window_import(kg[g0:g0 + cnt].contiguous(), limbs[g0 * 6:(g0 + cnt) * 6].contiguous(), g0=g0, count=cnt)
            parts.append(a.finalize()[g0:g0 + cnt])
    assert_bits_equal(torch.cat(parts).cpu().numpy(), ref)


@pytest.mark.parametrize("dtype,K,G", [(np.float64, 3, 16), (np.float64, 2, 3), (np.float32, 2, 16),
                                       (np.float32, 3, 1)])
@pytest.mark.parametrize("case", ["tiny_group", "late_large", "zeros", "one_window"])
def test_lean_single_window_checks(R, dtype, K, G, case):
    """The lean kernel (<= 16 groups) keeps a block only if every value is at
    or below the block's window k0 and every group it touched has a value AT
    k0; the cases below force each kind of fallback (and one that needs none).
    Bits must equal the oracle's either way."""
    rng = np.random.default_rng(G * 10 + K)
    n = (1 << 20) + 9
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = (rng.uniform(1, 2, n) * np.where(rng.random(n) < 0.5, -1, 1)).astype(dtype)
    if case == "tiny_group":  # group G-1 holds only values far below the others' window
        vals[keys == G - 1] *= 2.0 ** -60 if dtype == np.float64 else 2.0 ** -30
    elif case == "late_large":  # a value above the window late in every block
        vals[n - 3] = 2.0 ** 100 if dtype == np.float64 else 2.0 ** 40
        vals[n // 2] = -(2.0 ** 90) if dtype == np.float64 else -(2.0 ** 35)
    elif case == "zeros":
        vals[::7] = 0.0
    got = gpu_groupby(R, keys, vals, G, K)
    assert_bits_equal(got, oracle_groupby(keys, vals, G, K))


def test_lean_single_is_the_one_that_runs(R):
    keys, vals = synth.generate_chunked(1, 1 << 20, 16)
    R.timing_enable(True)
    R.timing_collect()
    gpu_groupby(R, keys, vals, 16, 3)
    names = R.timing_collect()
    R.timing_enable(False)
    assert "lean_single" in names and "onchip_accumulate" not in names


def test_host_entry_point_matches(R):
    keys, vals = synth.generate_chunked(1, (1 << 23) + 12345, 1024)
    kt, vt = torch.from_numpy(keys).pin_memory(), torch.from_numpy(vals).pin_memory()
    got = R.groupby_sum_host(kt, vt, 1024, 3).numpy()
    got_pageable = R.groupby_sum_host(torch.from_numpy(keys), torch.from_numpy(vals), 1024, 3).numpy()
    ref = gpu_groupby(R, keys, vals, 1024, 3)
    assert_bits_equal(got, ref)
    assert_bits_equal(got_pageable, ref)


def test_async_entry_point(R):
    keys, vals = synth.generate(0)
    ws = R.make_workspace(keys.size, 16, 3, R.F64)
    status = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    out = torch.empty(16, dtype=torch.float64, device="cuda")
    R.groupby_sum_async(dev(keys), dev(vals), 16, 3, out, ws, status)
    torch.cuda.synchronize()
    assert status.item() == 0
    assert_bits_equal(out.cpu().numpy(), oracle_groupby(keys, vals, 16, 3))
    bad = vals.copy()
    bad[3] = np.nan
    R.groupby_sum_async(dev(keys), dev(bad), 16, 3, out, ws, status)
    torch.cuda.synchronize()
    assert status.item() == R.EDOM


# ------------------------------------------------------- baseline witness (P-12)

def test_atomic_baseline_is_not_reproducible(R):
    base = [2.5e-16, 0.999999999999999, 2.5e-16]
    rng = np.random.default_rng(0)
    seen = set()
    G = 64
    vals0 = np.array(base * 20000)
    keys0 = np.repeat(np.arange(G, dtype=np.int32), vals0.size // G + 1)[: vals0.size]
    for t in range(20):
        p = rng.permutation(vals0.size)
        out = R.baseline_atomic_sum(dev(keys0[p]), dev(vals0[p]), G, variant=t % 2)
        torch.cuda.synchronize()
        seen.add(out.cpu().numpy().tobytes())
    assert len(seen) >= 2
    # the reproducible path gives one answer for all of them
    outs = {gpu_groupby(R, keys0[p], vals0[p], G, 2).tobytes()
            for p in (rng.permutation(vals0.size) for _ in range(4))}
    assert len(outs) == 1


def test_atomic_baseline_close_to_repro(R):
    keys, vals = synth.generate_chunked(1, 1 << 20, 1024)
    rep = gpu_groupby(R, keys, vals, 1024, 3)
    for variant in (0, 1, 3, 4):
        b = R.baseline_atomic_sum(dev(keys), dev(vals), 1024, variant=variant).cpu().numpy()
        np.testing.assert_allclose(b, rep, rtol=1e-9, atol=1e-6)


@pytest.mark.parametrize("n", [(1 << 20) + 3, 1001, 5])
def test_atomic_baseline_register_variant(R, n):
    # G <= 16: 16-byte loads with a scalar remainder (ragged n)
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 16, n, dtype=np.int32)
    vals = rng.uniform(-1, 1, n)
    rep = gpu_groupby(R, keys, vals, 16, 3)
    b = R.baseline_atomic_sum(dev(keys), dev(vals), 16, variant=2).cpu().numpy()
    np.testing.assert_allclose(b, rep, rtol=1e-9, atol=1e-9)


def test_atomic_baseline_heavy_hitters_on_zipf(R):
    # skewed keys: the heavy keys are summed per warp in shared memory, the
    # rest by global atomics; the sums agree with the reproducible ones
    rng = np.random.default_rng(7)
    G, n = 1 << 18, (1 << 21) + 1
    p = np.arange(1, G + 1, dtype=np.float64) ** -1.1
    keys = np.minimum(np.searchsorted(np.cumsum(p / p.sum()), rng.random(n)), G - 1).astype(np.int32)
    vals = rng.uniform(-1, 1, n)
    rep = gpu_groupby(R, keys, vals, G, 3)
    b = R.baseline_atomic_sum(dev(keys), dev(vals), G, variant=4).cpu().numpy()
    np.testing.assert_allclose(b, rep, rtol=1e-9, atol=1e-9)


# ------------------------------------------------- partitioned path (row a5)

@pytest.fixture(params=[1, 2], ids=["sweep", "segmented"])
def partitioned(R, request):
    """Force the partitioned path: 1 = the two-pass sweep (k_sweep.cu; beyond
    its 256 partitions the segmented passes), 2 = the segmented radix passes
    (k_partition.cu)."""
    R.set_path_override(request.param)
    yield request.param
    R.set_path_override(-1)


PART_CASES = [
    (np.float64, 3, 1, 30001, 20),
    (np.float64, 3, 1024, 200003, 20),
    (np.float64, 3, 5000, 300007, 40),
    (np.float64, 2, 70000, 500000, 60),
    (np.float32, 2, 3000, 400001, 10),
    (np.float32, 1, 40000, 300000, 30),
    (np.float64, 4, 2049, 100000, 200),
    # partition-pass plans (k_partition.cu make_plan): P = ceil(G / 1024)
    (np.float64, 3, (1 << 18) + 5, 600011, 30),   # P = 257: binary64 one wide pass (512 digits)
    (np.float64, 2, (1 << 20) - 3, 700001, 20),   # P = 1024: binary64 one wide pass (1024 digits)
    (np.float64, 2, (1 << 21) + 3, 500003, 20),   # P = 2049: binary64 two passes (6 + 6)
    (np.float32, 2, (1 << 19) + 1, 600001, 20),   # P = 513: binary32 one wide pass (1024 digits)
    (np.float32, 2, (1 << 21) + 7, 500003, 10),   # P = 2049: binary32 two passes (6 + 6)
]


@pytest.mark.parametrize("dtype,K,G,n,spread", PART_CASES)
def test_partitioned_forced_matches_oracle(R, partitioned, dtype, K, G, n, spread):
    rng = np.random.default_rng(7 * n + G)
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = mixed_values(rng, n, dtype, spread)
    got = gpu_groupby(R, keys, vals, G, K)
    assert R.last_path() == (2 if partitioned == 2 or G > R.sweep_max_groups(K, dtype_code(dtype)) else 1)
    assert_bits_equal(got, oracle_groupby(keys, vals, G, K))


@pytest.mark.parametrize("G", ["cap+1", 1 << 17, (1 << 20) + 5])
def test_partitioned_auto_above_onchip_capacity(R, G):
    # just above the on-chip table's capacity: the two-pass sweep (path 1);
    # beyond the sweep's 256 partitions: segmented radix passes (path 2)
    if G == "cap+1":
        G = R.onchip_max_groups(3, R.F64) + 1
    rng = np.random.default_rng(G)
    n = 1 << 20
    keys = rng.integers(0, G, n, dtype=np.int32)
    vals = mixed_values(rng, n, np.float64, 25)
    got = gpu_groupby(R, keys, vals, G, 3)
    assert R.last_path() == (1 if G <= (1 << 20) else 2)
    assert_bits_equal(got, oracle_groupby(keys, vals, G, 3))


def test_partitioned_skew_multi_item_partitions(R, partitioned):
    # Zipf over 2^16 groups: the first partitions hold many work items of 2^16 rows
    keys, vals = synth.generate_chunked(3, 1 << 21, 1 << 16)
    got = gpu_groupby(R, keys, vals, 1 << 16, 2)
    assert_bits_equal(got, oracle_groupby(keys, vals, 1 << 16, 2))


def test_partitioned_empty_partitions_and_groups(R, partitioned):
    G = 1 << 20
    rng = np.random.default_rng(3)
    keys = np.concatenate([rng.integers(5000, 6000, 50000), rng.integers(900000, 900100, 50000)]).astype(np.int32)
    vals = mixed_values(rng, keys.size, np.float64, 30)
    got = gpu_groupby(R, keys, vals, G, 3)
    assert_bits_equal(got, oracle_groupby(keys, vals, G, 3))
    out = gpu_groupby(R, np.zeros(0, np.int32), np.zeros(0), G, 3)
    assert out.tobytes() == np.zeros(G).tobytes()


def test_partitioned_accumulator_deposits(R, partitioned):
    G = 9000
    rng = np.random.default_rng(4)
    keys = rng.integers(0, G, 600000, dtype=np.int32)
    vals = mixed_values(rng, keys.size, np.float64, 40)
    a = R.Accumulator(G, 3, R.F64)
    for c0, c1 in ((0, 100000), (100000, 100001), (100001, 600000)):
        a.deposit(dev(keys[c0:c1]), dev(vals[c0:c1]))
    rc, ref, st = O.groupby_sum(keys, vals, G, 3, with_state=True)
    assert_bits_equal(a.finalize().cpu().numpy(), ref)
    assert a.export().cpu().numpy().reshape(G, 6).tobytes() == st.tobytes()


def test_partitioned_errors(R, partitioned):
    keys = np.zeros(100000, np.int32)
    vals = np.ones(100000)
    keys[99999] = 70000
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 5000, 3)
    assert ei.value.status == R.EKEY
    keys[99999] = 1
    vals[5] = np.nan
    with pytest.raises(R.ReproError) as ei:
        gpu_groupby(R, keys, vals, 5000, 3)
    assert ei.value.status == R.EDOM


@pytest.mark.parametrize("dtype,K,G,n", [(np.float64, 3, 1 << 16, (1 << 21) + 3), (np.float32, 2, 1 << 20, 1 << 22),
                                         (np.float64, 2, 5000, 1 << 20)])
def test_partitioned_heavy_partition_summed_in_place(R, dtype, K, G, n):
    # Zipf keys: partition 0 holds more than n/2 of the rows, so the plan
    # sums it in place from the original columns instead of scattering it
    keys, _ = synth.generate_chunked(3, n, G)
    rng = np.random.default_rng(G)
    vals = mixed_values(rng, n, dtype, 30)
    bad = keys.copy()
    R.set_path_override(1)
    try:
        got = gpu_groupby(R, keys, vals, G, K)
        assert R.last_path() == 1
        assert_bits_equal(got, oracle_groupby(keys, vals, G, K))
        bad[n // 3] = G + 5  # an out-of-range key inside the heavy partition's key range is still EKEY
        with pytest.raises(R.ReproError) as e:
            gpu_groupby(R, bad, vals, G, K)
        assert e.value.status == R.EKEY
    finally:
        R.set_path_override(-1)
