"""Oracle pins for the multi-column GroupBy (repro_groupby_sum_multi): the
config-4 projection of reading A-15 against exact rational
arithmetic rounded once per operation, COUNT against a loop, and the
multi-column call against one single-column call per column."""
from fractions import Fraction

import numpy as np

import oracle as O
from inputs import synth


def rn64(q: Fraction) -> float:
    """Round an exact rational to the nearest binary64 (ties to even) --
    float(Fraction) is correctly rounded in CPython."""
    return float(q)


def test_q1_projection_is_one_rounding_per_operation():
    rng = np.random.default_rng(4)
    price = (90000 + rng.integers(0, 10410001, 2000)) / 100.0
    disc = rng.integers(0, 11, 2000) / 100.0
    tax = rng.integers(0, 9, 2000) / 100.0
    dp, ch = O.q1_project(price, disc, tax)
    for i in range(2000):
        d1 = rn64(1 - Fraction(disc[i]))
        want_dp = rn64(Fraction(price[i]) * Fraction(d1))
        t1 = rn64(1 + Fraction(tax[i]))
        want_ch = rn64(Fraction(want_dp) * Fraction(t1))
        assert dp[i] == want_dp and ch[i] == want_ch, i


def test_q1_projection_differs_from_fused_evaluation_somewhere():
    # the reading matters: evaluating price*(1-disc)*(1+tax) exactly and
    # rounding once gives other bits for some rows (so a GPU path that
    # contracted to FMA would be caught by the parity tests)
    keys, (qty, price, disc, tax) = synth.generate(4, n=20000)
    dp, ch = O.q1_project(price, disc, tax)
    diff = 0
    for i in range(20000):
        exact = Fraction(price[i]) * (1 - Fraction(disc[i])) * (1 + Fraction(tax[i]))
        diff += rn64(exact) != ch[i]
    assert diff > 0


def test_multi_counts_and_columns_equal_single_calls():
    rng = np.random.default_rng(9)
    n, G = 30000, 37
    keys = rng.integers(0, G, n).astype(np.int32)
    cols = [rng.standard_normal(n) * 2.0 ** rng.integers(-30, 30, n) for _ in range(3)]
    rc, outs, counts = O.groupby_sum_multi(keys, cols, G, 3)
    assert rc == O.OK
    loop = np.zeros(G, np.int64)
    for k in keys:
        loop[k] += 1
    assert np.array_equal(counts, loop)
    for c, o in zip(cols, outs):
        rc1, o1 = O.groupby_sum(keys, c, G, 3)
        assert rc1 == O.OK and o1.tobytes() == o.tobytes()


def test_multi_q1_equals_single_calls_on_projected_columns():
    keys, (qty, price, disc, tax) = synth.generate(4, n=40000)
    rc, outs, counts = O.groupby_sum_multi(keys, [qty, price, disc, tax], 4, 3, proj=1)
    assert rc == O.OK and len(outs) == 4 and counts.sum() == 40000
    dp, ch = O.q1_project(price, disc, tax)
    for c, o in zip([qty, price, dp, ch], outs):
        assert O.groupby_sum(keys, c, 4, 3)[1].tobytes() == o.tobytes()
    # qty is integral: its reproducible sum is the exact integer sum
    assert np.array_equal(outs[0], np.bincount(keys, weights=qty, minlength=4))


def test_multi_error_precedence():
    keys = np.array([0, 1, 5], np.int32)
    a = np.array([1.0, np.nan, 2.0])
    b = np.array([1.0, 2.0, 3.0])
    rc, _, _ = O.groupby_sum_multi(keys, [a, b], 3, 2)
    assert rc == O.EKEY
    rc, _, _ = O.groupby_sum_multi(np.array([0, 1, 2], np.int32), [b, a], 3, 2)
    assert rc == O.EDOM


def test_moments_exact_on_integer_data():
    # small integers: the reproducible sums are exact, so AVG / VARIANCE follow
    # from exact rationals rounded once per operation
    rng = np.random.default_rng(12)
    keys = rng.integers(0, 5, 3000).astype(np.int32)
    x = rng.integers(-1000, 1000, 3000).astype(np.float64)
    rc, m = O.groupby_moments(keys, x, 5, 3)
    assert rc == O.OK
    for g in range(5):
        xs = [Fraction(int(v)) for v in x[keys == g]]
        c = len(xs)
        s, q = sum(xs), sum(v * v for v in xs)
        assert m["sum"][g] == float(s) and m["count"][g] == c
        assert m["avg"][g] == rn64(s / Fraction(c))
        t = Fraction(float(q)) - Fraction(rn64(Fraction(float(s)) * Fraction(float(s)) / c))
        want_var = max(0.0, rn64(Fraction(rn64(t)) / (c - 1)))
        assert m["var"][g] == want_var
        assert m["stddev"][g] == np.sqrt(want_var)


def test_moments_special_counts():
    keys = np.array([0, 1, 1], np.int32)
    x = np.array([2.5, -1.0, 3.0])
    rc, m = O.groupby_moments(keys, x, 3, 2)
    assert rc == O.OK
    assert m["count"].tolist() == [1, 2, 0]
    assert m["avg"].tolist() == [2.5, 1.0, 0.0]
    assert m["var"].tolist() == [0.0, 8.0, 0.0]  # ((9+1) - 4/2) / 1


def test_sparse_keys_dense_domain_equals_dense_groupby():
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 50, 4000)
    vals = rng.standard_normal(4000)
    rc, uk, out = O.groupby_sum_sparse(keys, vals, 3)
    assert rc == O.OK and np.array_equal(uk, np.unique(keys))
    rc2, dense = O.groupby_sum(keys.astype(np.int32), vals, 50, 3)
    assert out.tobytes() == dense[uk].tobytes()


def test_sparse_keys_reserved_and_empty():
    assert O.groupby_sum_sparse(np.array([3, O.INT64_MIN]), np.array([1.0, 2.0]), 2)[0] == O.EKEY
    rc, uk, out = O.groupby_sum_sparse(np.zeros(0, np.int64), np.zeros(0), 2)
    assert rc == O.OK and uk.size == 0 and out.size == 0
