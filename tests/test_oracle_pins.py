"""Pins for the CPU oracle (``oracle/``) against what the paper and the
mathematics fix -- never against the oracle itself.

Pins:
  P-1  three-row example of PAPER.md:111-118, every permutation
  P-2  half-precision EFT example, PAPER.md:527-532
  P-3  toy m=3 EFT example, PAPER.md:543-545
  P-4  carry example, PAPER.md:647-651
  P-5  toy-format brute force: permutation invariance of Alg. 1 (and its
       failure under the literal RNE / 2^W readings)
  P-6  exact-rational integer-digit closed form (tests/exact_ref.py)
  P-7  permutation / chunking / merge-tree / thread-count invariance
  P-8  state exactness on config-0-shaped data
  P-9  Table 3 bound formulas, PAPER.md:1318-1337
  P-10 special cases with textbook answers
  P-11 error bound on the represented value, incl. adversarial input
  plus the hand-derived toy trace of PAPER.md:711-731 and error codes.
"""
import itertools
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import exact_ref as X
import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
F32, F64 = O.F32, O.F64
BITS = {F64: 64, F32: 32}


def bits64(x):
    return np.float64(x).view(np.uint64).item()


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# --------------------------------------------------------------------------
# primitives: ufp / ulp / EFT / rounding
# --------------------------------------------------------------------------

def test_ufp_ulp_spec_examples():
    assert O.ufp(1.5) == 1.0
    assert O.ufp(-6.5) == 4.0
    assert O.ufp(0.15625) == 0.125
    assert O.ulp(O.params(F64, 1), 1.0) == 2.0 ** -52
    assert O.ulp(O.params(m=4, W=2, K=1), 27.0) == 1.0
    assert O.ulp(O.params(F32, 1), 0.5) == 2.0 ** -24


def test_eft_half_precision_example():
    # 26.046875 (+) 2.8125 = 28.859375 exactly in m = 10
    p = O.params(m=10, W=8, K=1, emin=-14, emax=15)
    assert O.fadd(p, 26.046875, 2.8125) == 28.859375
    assert 26.046875 == 1667 * 2.0 ** -6 and 2.8125 == 180 * 2.0 ** -6


def test_eft_toy_m3_example():
    # PAPER.md:543-545 with the definition q = (a (+) b) (-) a (A-13)
    p = O.params(m=3, W=1, K=1, emin=-20, emax=20)
    q, r = O.eft(p, 1.25, 0.40625)
    assert (q, r) == (0.375, 0.03125)
    assert q + r == 0.40625  # error-free


def test_eft_zero():
    p = O.params(F64, 1)
    assert O.eft(p, 1.5, 0.0) == (0.0, 0.0)


def test_toy_rounding_matches_binary32_hardware():
    # The toy rounding path with m = 23 must be binary32 round-to-nearest-even.
    rng = np.random.default_rng(1)
    p = O.params(m=23, W=18, K=1, emin=-126, emax=127)
    for _ in range(2000):
        a = np.float32(rng.standard_normal() * 2.0 ** rng.integers(-8, 8))
        b = np.float32(rng.standard_normal() * 2.0 ** rng.integers(-8, 8))
        assert O.fadd(p, float(a), float(b)) == float(a + b)


def test_toy_lsb_force_matches_bit_operation():
    rng = np.random.default_rng(2)
    p64 = O.params(F64, 1)
    t64 = O.params(m=52, W=40, K=1, emin=-1022, emax=1023)
    p32 = O.params(F32, 1)
    t32 = O.params(m=23, W=18, K=1, emin=-126, emax=127)
    xs = list(rng.standard_normal(500) * 2.0 ** rng.integers(-30, 30, 500)) + [0.0, -0.0, 5e-324]
    for x in xs:
        u = np.float64(x).view(np.uint64) | np.uint64(1)
        assert bits64(O.lsb_force(p64, x)) == u.item()
        assert bits64(O.lsb_force(t64, x)) == u.item()
        f = np.float32(x)
        g = (f.view(np.uint32) | np.uint32(1)).view(np.float32)
        assert O.lsb_force(p32, float(f)) == float(g)
        assert O.lsb_force(t32, float(f)) == float(g)


def test_carry_examples():
    # S = 1.84 ufp -> d = 1 -> 1.59 ufp, C += 1 (grid of 1/100 in units of 2^-?):
    # use binary64 values 1.84 * 2^10 and 1.40 * 2^10
    p = O.params(F64, 1)
    S, C = O.carry(p, 1.84 * 1024, 0.0)
    assert C == 1.0 and S == 1.84 * 1024 - 256 and 1.5 * 1024 <= S < 1.75 * 1024
    S, C = O.carry(p, 1.40 * 1024, 0.0)
    assert C == -1.0 and S == 1.40 * 1024 + 256
    S, C = O.carry(p, 1.6 * 1024, 3.0)
    assert (S, C) == (1.6 * 1024, 3.0)


def test_init_spec_examples():
    st = O.init(O.params(m=4, W=2, K=2, f=4))
    assert st.S == [24.0, 6.0] and st.C == [0.0, 0.0]
    st = O.init(O.params(F64, 1))
    assert st.S == [1.5]
    p = O.params(F32, 3)
    p.f = 36
    assert O.init(p).S == [1.5 * 2.0 ** 36, 1.5 * 2.0 ** 18, 1.5]


def test_finalize_spec_examples():
    p = O.params(m=4, W=2, K=1, f=4)
    assert O.finalize(p, O.State([27.0], [0.0])) == 3.0
    assert O.finalize(p, O.State([27.0], [1.0])) == 7.0
    assert O.finalize(p, O.init(p)) == 0.0


# --------------------------------------------------------------------------
# hand-derived toy trace of PAPER.md:711-731 (reading A-13: result 12)
# --------------------------------------------------------------------------

def test_toy_trace_hand_derived():
    rows = read_golden("toy_trace.txt")
    assert rows[0] == ["step", "S1", "S2", "C1", "C2"]
    p = O.params(m=4, W=2, K=2, f=4, emin=-30, emax=30)
    st = O.init(p)
    for row in rows[1:]:
        if row[0] == "Q":
            assert O.finalize(p, st) == float(row[1])
            continue
        if row[0] != "init":
            assert O.deposit(p, st, float(row[0])) == O.OK
        assert st.S == [float(row[1]), float(row[2])]
        assert st.C == [float(row[3]), float(row[4])]


def test_toy_trace_2W_threshold_gives_paper_prose_value():
    # The prose value 14 is what a 2^W threshold produces; kept as a
    # documentation pin of reading A-2 (the 2^W reading is not reproducible, see P-5).
    p = O.params(m=4, W=2, K=2, f=4, emin=-30, emax=30, thr_shift=2)
    st = O.deposit_all(p, [1.3125, 9, 4.25])
    assert O.finalize(p, st) == 14.0


# --------------------------------------------------------------------------
# P-1 three-row example
# --------------------------------------------------------------------------

THREE = [2.5e-16, 0.999999999999999, 2.5e-16]


def test_three_row_plain_sums_differ():
    g = {r[0]: int(r[1], 16) for r in read_golden("three_row.txt")}
    p = O.params(F64, 1)
    assert bits64(O.plain_sum(p, [THREE[0], THREE[1], THREE[2]])) == g["plain_123"]
    assert bits64(O.plain_sum(p, [THREE[0], THREE[2], THREE[1]])) == g["plain_132"]
    assert g["plain_123"] != g["plain_132"]  # the paper's non-reproducibility
    assert bits64(float(X.exact_sum(THREE))) == g["exact_rn"]


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_three_row_every_permutation_same_bits(K):
    g = {r[0]: int(r[1], 16) for r in read_golden("three_row.txt")}
    p = O.params(F64, K)
    seen = set()
    for perm in itertools.permutations(THREE):
        st = O.deposit_all(p, perm)
        seen.add((st.key(), bits64(O.finalize(p, st))))
    assert len(seen) == 1
    (_, q), = seen
    assert q == g[f"repro_K{K}"]


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_three_row_golden_is_closed_form(K):
    g = {r[0]: int(r[1], 16) for r in read_golden("three_row.txt")}
    ktop, T = X.state_closed_form(THREE, K, 64)
    assert bits64(X.finalize_closed_form(ktop, T, 64)) == g[f"repro_K{K}"]


def test_three_row_literal_rne_is_order_dependent():
    # Reading A-1 is needed: the literal RNE extraction gives two results at K=2.
    p = O.params(F64, 2, ties_away=False)
    res = set()
    for perm in itertools.permutations(THREE):
        st = O.deposit_all(p, perm)
        res.add(bits64(O.finalize(p, st)))
    assert len(res) == 2


# --------------------------------------------------------------------------
# P-5 toy brute force
# --------------------------------------------------------------------------

def _toy_values():
    vals = []
    for e in range(-3, 4):
        for mant in range(16, 32):
            for s in (1, -1):
                vals.append(s * mant * 2.0 ** (e - 4))
    return vals


def _count_non_invariant(p, trials, size_choices, seed):
    rng = random.Random(seed)
    vals = _toy_values()
    bad = 0
    for _ in range(trials):
        ms = [rng.choice(vals) for _ in range(rng.choice(size_choices))]
        outs = set()
        for perm in set(itertools.permutations(ms)):
            st = O.deposit_all(p, perm)
            outs.add((st.key(), O.finalize(p, st)))
        bad += len(outs) > 1
    return bad


def test_toy_bruteforce_permutation_invariant():
    p = O.params(m=4, W=2, K=2, f=0, emin=-40, emax=30)
    assert _count_non_invariant(p, 600, (3, 4), seed=5) == 0


def test_toy_bruteforce_literal_rne_fails():
    p = O.params(m=4, W=2, K=2, f=0, emin=-40, emax=30, ties_away=False)
    assert _count_non_invariant(p, 300, (3, 4), seed=6) > 0


def test_toy_bruteforce_2W_threshold_fails():
    p = O.params(m=4, W=2, K=2, f=0, emin=-40, emax=30, thr_shift=2)
    assert _count_non_invariant(p, 300, (3, 4), seed=7) > 0


def test_toy_bruteforce_against_exact_bound():
    # every toy result is within the represented-value bound n ulp_K / 2 of the exact sum
    p = O.params(m=4, W=2, K=2, f=0, emin=-40, emax=30)
    rng = random.Random(8)
    vals = _toy_values()
    for _ in range(400):
        ms = [rng.choice(vals) for _ in range(rng.choice((2, 3, 5)))]
        st = O.deposit_all(p, ms)
        V = sum(Fraction(S) - Fraction(3, 2) * Fraction(O.ufp(S)) + Fraction(C) * Fraction(O.ufp(S)) / 4
                for S, C in zip(st.S, st.C))
        uK = Fraction(O.ulp(p, st.S[-1]))
        assert abs(V - X.exact_sum(ms)) <= len(ms) * uK / 2


# --------------------------------------------------------------------------
# P-6 closed form (exact rationals) == oracle state and result, bit for bit
# --------------------------------------------------------------------------

def _random_values(rng, n, bits, spread):
    out = []
    for _ in range(n):
        e = int(rng.integers(-spread, spread + 1))
        v = rng.uniform(1, 2) * 2.0 ** e * (1 if rng.random() < 0.5 else -1)
        if rng.random() < 0.05:
            v = 0.0
        out.append(float(np.float32(v)) if bits == 32 else v)
    return out


@pytest.mark.parametrize("bits,K,spread", [(64, 1, 30), (64, 2, 30), (64, 3, 60), (64, 4, 90),
                                           (64, 3, 200), (32, 1, 10), (32, 2, 20), (32, 3, 40),
                                           (32, 4, 60)])
def test_closed_form_equals_oracle(bits, K, spread):
    rng = np.random.default_rng(100 + bits + K + spread)
    dtype = F64 if bits == 64 else F32
    p = O.params(dtype, K)
    for trial in range(40):
        vals = _random_values(rng, int(rng.integers(1, 40)), bits, spread)
        st = O.deposit_all(p, vals)
        ktop, T = X.state_closed_form(vals, K, bits)
        S, C = X.canonical_SC(ktop, T, bits)
        assert st.S == S and st.C == C, (vals, st, S, C)
        q = O.finalize(p, st)
        assert bits64(q) == bits64(X.finalize_closed_form(ktop, T, bits))


def test_closed_form_digits_above_kstar_are_zero():
    # digits of a value at levels above its own k* vanish (needed by A-2):
    for bits in (64, 32):
        m, W, _ = X.FMT[bits]
        rng = np.random.default_rng(bits)
        for v in _random_values(rng, 300, bits, 100 if bits == 64 else 30):
            k = X.kstar(v, bits)
            for j in range(k + 1, k + 4):
                u = Fraction(2) ** (W * j - m)
                assert X.round_half_away(Fraction(v) / u) == 0


# --------------------------------------------------------------------------
# P-7 invariances (AC1-3 SPEC.md:551-553)
# --------------------------------------------------------------------------

def _gb_inputs(seed, n, G, dtype):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, G, n, dtype=np.int32)
    e = rng.integers(-20, 21, n)
    v = (rng.uniform(1, 2, n) * np.exp2(e) * rng.choice([-1, 1], n))
    return keys, v.astype(np.float64 if dtype == F64 else np.float32)


@pytest.mark.parametrize("dtype,K", [(F64, 3), (F64, 2), (F32, 2), (F32, 4)])
def test_groupby_thread_and_mode_invariance(dtype, K):
    keys, vals = _gb_inputs(11, 20000, 37, dtype)
    ref = O.groupby_sum(keys, vals, 37, K, threads=1, mode=1, with_state=True)
    assert ref[0] == O.OK
    for threads in (2, 3, 8):
        for mode in (1, 2):
            got = O.groupby_sum(keys, vals, 37, K, threads=threads, mode=mode, with_state=True)
            assert got[0] == O.OK
            assert got[1].tobytes() == ref[1].tobytes()
            assert got[2].tobytes() == ref[2].tobytes()


@pytest.mark.parametrize("dtype,K", [(F64, 3), (F32, 2)])
def test_groupby_permutation_invariance(dtype, K):
    keys, vals = _gb_inputs(12, 30000, 16, dtype)
    ref = O.groupby_sum(keys, vals, 16, K, with_state=True)
    rng = np.random.default_rng(3)
    for _ in range(3):
        perm = rng.permutation(keys.size)
        got = O.groupby_sum(keys[perm], vals[perm], 16, K, with_state=True)
        assert got[1].tobytes() == ref[1].tobytes() and got[2].tobytes() == ref[2].tobytes()


def test_merge_tree_and_chunking_invariance():
    rng = np.random.default_rng(21)
    for dtype, K in ((F64, 3), (F32, 2), (F64, 1)):
        p = O.params(dtype, K)
        vals = _random_values(rng, 400, BITS[dtype], 40 if dtype == F64 else 12)
        whole = O.deposit_all(p, vals)
        for trial in range(5):
            cuts = sorted(rng.choice(np.arange(1, len(vals)), size=7, replace=False))
            parts = [O.deposit_all(p, c) for c in np.split(np.array(vals), cuts)]
            order = list(rng.permutation(len(parts)))
            while len(order) > 1:  # random merge tree
                i, j = sorted(rng.choice(len(order), size=2, replace=False))
                a, b = parts[order[i]], parts[order[j]]
                assert O.merge(p, a, b) == O.OK
                order.pop(j)
            merged = parts[order[0]]
            assert merged.key() == whole.key()


def test_merge_monoid_laws():
    rng = np.random.default_rng(22)
    for dtype, K in ((F64, 3), (F32, 2)):
        p = O.params(dtype, K)
        for _ in range(20):
            a, b, c = (O.deposit_all(p, _random_values(rng, 30, BITS[dtype], 50)) for _ in range(3))
            # identity
            x = O.State(list(a.S), list(a.C)); O.merge(p, x, O.init(p)); assert x.key() == a.key()
            y = O.init(p); O.merge(p, y, a); assert y.key() == a.key()
            # commutativity
            ab = O.State(list(a.S), list(a.C)); O.merge(p, ab, b)
            ba = O.State(list(b.S), list(b.C)); O.merge(p, ba, a)
            assert ab.key() == ba.key()
            # associativity
            ab_c = O.State(list(ab.S), list(ab.C)); O.merge(p, ab_c, c)
            bc = O.State(list(b.S), list(b.C)); O.merge(p, bc, c)
            a_bc = O.State(list(a.S), list(a.C)); O.merge(p, a_bc, bc)
            assert ab_c.key() == a_bc.key()


# --------------------------------------------------------------------------
# P-8 state exactness for config-0-shaped fp64 data at K=3
# --------------------------------------------------------------------------

def test_config0_shape_state_is_exact():
    rng = np.random.default_rng(30)
    p = O.params(F64, 3)
    for _ in range(20):
        n = 64
        mant = rng.integers(0, 2 ** 52, n, dtype=np.uint64)
        e = rng.integers(-20, 21, n)
        sign = rng.integers(0, 2, n)
        bitsv = (sign.astype(np.uint64) << np.uint64(63)) | ((e + 1023).astype(np.uint64) << np.uint64(52)) | mant
        vals = [float(x) for x in bitsv.view(np.float64)]
        st = O.deposit_all(p, vals)
        V = sum(Fraction(S) - Fraction(3, 2) * Fraction(O.ufp(S)) + Fraction(C) * Fraction(O.ufp(S)) / 4
                for S, C in zip(st.S, st.C))
        assert V == X.exact_sum(vals)


# --------------------------------------------------------------------------
# P-9 Table 3: the bound formulas with eps = 2^-53
# --------------------------------------------------------------------------

def e_conv(n, sum_abs, eps=2.0 ** -53):
    return (n - 1) * eps * sum_abs


def e_rsum(n, L, W, maxabs):
    return n * 2.0 ** ((1 - L) * W - 1) * maxabs


def test_table3_formula_values():
    mean = {"U": 1.5, "E": 1.0}
    mx = {"U": 2.0, "E": 22.0}
    for row, n, dist, val in read_golden("table3.txt"):
        n, val = int(n), float(val)
        if row == "conv":
            got = e_conv(n, mean[dist] * n)
        else:
            got = e_rsum(n, int(row[1]), 40, mx[dist])
        assert float(f"{got:.1e}") == val, (row, n, dist, got)


# --------------------------------------------------------------------------
# P-10 special cases
# --------------------------------------------------------------------------

def test_single_value_round_trips():
    rng = np.random.default_rng(40)
    p = O.params(F64, 3)
    for _ in range(300):
        v = rng.uniform(1, 2) * 2.0 ** int(rng.integers(-80, 987)) * rng.choice([-1, 1])
        assert O.finalize(p, O.deposit_all(p, [v])) == v
    p32 = O.params(F32, 3)
    for _ in range(300):
        v = float(np.float32(rng.uniform(1, 2) * 2.0 ** int(rng.integers(-36, 120))))
        assert O.finalize(p32, O.deposit_all(p32, [v])) == v


def test_cancellation_gives_positive_zero():
    for dtype, K in ((F64, 3), (F32, 2), (F64, 1)):
        p = O.params(dtype, K)
        for x in (1.0, 3.25e-7, -12345.5, 2.0 ** 60):
            q = O.finalize(p, O.deposit_all(p, [x, -x]))
            assert q == 0.0 and math.copysign(1.0, q) == 1.0


def test_million_ones_k2():
    keys = np.zeros(10 ** 6, dtype=np.int32)
    rc, out = O.groupby_sum(keys, np.ones(10 ** 6), 1, 2)
    assert rc == O.OK and out[0] == 1000000.0


def test_empty_input_and_empty_groups():
    rc, out = O.groupby_sum(np.zeros(0, np.int32), np.zeros(0), 5, 3)
    assert rc == O.OK and out.tobytes() == np.zeros(5).tobytes()
    rc, out = O.groupby_sum(np.array([3], np.int32), np.array([2.5]), 5, 3)
    assert rc == O.OK and list(out) == [0, 0, 0, 2.5, 0]
    assert np.signbit(out).sum() == 0


# --------------------------------------------------------------------------
# P-11 error bound on the represented value (reading A-12)
# --------------------------------------------------------------------------

def _V(st):
    return sum(Fraction(S) - Fraction(3, 2) * Fraction(O.ufp(S)) + Fraction(C) * Fraction(O.ufp(S)) / 4
               for S, C in zip(st.S, st.C))


@pytest.mark.parametrize("dtype,K", [(F64, 1), (F64, 2), (F64, 3), (F32, 1), (F32, 2), (F32, 3)])
def test_bound_on_random_inputs(dtype, K):
    rng = np.random.default_rng(50 + K + dtype)
    p = O.params(dtype, K)
    eps = 2.0 ** -53 if dtype == F64 else 2.0 ** -24
    for _ in range(40):
        vals = _random_values(rng, int(rng.integers(1, 60)), BITS[dtype], 30 if dtype == F64 else 10)
        st = O.deposit_all(p, vals)
        V = _V(st)
        uK = Fraction(O.ulp(p, st.S[-1]))
        assert abs(V - X.exact_sum(vals)) <= len(vals) * uK / 2
        # output: K roundings of t_l plus K-1 chain additions
        q = O.finalize(p, st)
        ts = [abs(Fraction(S) - Fraction(3, 2) * Fraction(O.ufp(S)) + Fraction(C) * Fraction(O.ufp(S)) / 4)
              for S, C in zip(st.S, st.C)]
        assert abs(Fraction(q) - V) <= Fraction(2 * K) * Fraction(eps) * sum(ts) * Fraction(1001, 1000)


def test_bound_adversarial_exceeds_printed_bound_by_about_2():
    # b = 2^-13 + 2^-53 - 2^-65 drops ~2^-53 per row at K=2 (reading A-12):
    b = 2.0 ** -13 + 2.0 ** -53 - 2.0 ** -65
    n = 1000
    p = O.params(F64, 2)
    st = O.deposit_all(p, [b] * n)
    err = abs(_V(st) - X.exact_sum([b] * n))
    printed = Fraction(e_rsum(n, 2, 40, b))
    assert err > printed                                   # the printed bound is exceeded
    assert float(err / printed) == pytest.approx(2.0, rel=1e-3)
    assert err <= n * Fraction(O.ulp(p, st.S[-1])) / 2      # the state bound holds


# --------------------------------------------------------------------------
# error codes and their precedence (reading A-10)
# --------------------------------------------------------------------------

def test_error_codes_and_precedence():
    k = np.array([0, 1, 2], np.int32)
    assert O.groupby_sum(k, np.array([1.0, np.nan, 2.0]), 3, 3)[0] == O.EDOM
    assert O.groupby_sum(k, np.array([1.0, np.inf, 2.0]), 3, 3)[0] == O.EDOM
    assert O.groupby_sum(np.array([0, 3, 1], np.int32), np.array([1.0, 1.0, 2.0]), 3, 3)[0] == O.EKEY
    assert O.groupby_sum(np.array([0, -1, 1], np.int32), np.array([1.0, 1.0, 2.0]), 3, 3)[0] == O.EKEY
    assert O.groupby_sum(k, np.array([1.0, 2.0 ** 987, 2.0]), 3, 3)[0] == O.ERANGE
    assert O.groupby_sum(k, np.array([1.0, 2.0 ** 986, 2.0]), 3, 3)[0] == O.OK
    assert O.groupby_sum(k, np.array([1.0, 2.0 ** 120, 2.0], np.float32), 3, 2)[0] == O.ERANGE
    assert O.groupby_sum(k, np.array([1.0, 2.0 ** 119, 2.0], np.float32), 3, 2)[0] == O.OK
    # precedence EKEY > EDOM > ERANGE regardless of row order
    kk = np.array([0, 5, 1, 2], np.int32)
    vv = np.array([2.0 ** 1000, 1.0, np.nan, 1.0])
    for perm in itertools.permutations(range(4)):
        perm = list(perm)
        assert O.groupby_sum(kk[perm], vv[perm], 3, 3)[0] == O.EKEY
    kk = np.array([0, 1, 2], np.int32)
    vv = np.array([2.0 ** 1000, np.nan, 1.0])
    assert O.groupby_sum(kk, vv, 3, 3)[0] == O.EDOM
    assert O.groupby_sum(kk, np.array([1.0, 2.0, 3.0]), 0, 3)[0] == O.EINVAL
    assert O.groupby_sum(kk, np.array([1.0, 2.0, 3.0]), 3, 5)[0] == O.EINVAL


def test_select_matches_full():
    keys, vals = _gb_inputs(60, 50000, 300, F64)
    rc, out, st = O.groupby_sum(keys, vals, 300, 3, with_state=True)
    sel = np.array([0, 7, 299, 150, 42], np.int32)
    rc2, out2, st2 = O.groupby_sum_select(keys, vals, 300, 3, sel, with_state=True)
    assert rc == rc2 == O.OK
    assert out2.tobytes() == out[sel].tobytes() and st2.tobytes() == st[sel].tobytes()


def test_groupby_matches_closed_form_per_group():
    for dtype, K in ((F64, 3), (F32, 2)):
        keys, vals = _gb_inputs(70, 3000, 9, dtype)
        rc, out = O.groupby_sum(keys, vals, 9, K)
        for g in range(9):
            v = [float(x) for x in vals[keys == g]]
            ktop, T = X.state_closed_form(v, K, BITS[dtype])
            assert bits64(float(out[g])) == bits64(X.finalize_closed_form(ktop, T, BITS[dtype]))


# --------------------------------------------------------------------------
# edge values: window thresholds, subnormals, signed zeros, half-unit ties
# (Alg. 1 line 3 PAPER.md:660; readings A-1, A-9, A-11), pinned against the
# exact-rational closed form
# --------------------------------------------------------------------------

import edge_values as EV  # noqa: E402


@pytest.mark.parametrize("bits,K", [(64, 2), (64, 3), (32, 2), (32, 3)])
def test_edge_values_closed_form(bits, K):
    rng = np.random.default_rng(900 + bits + K)
    dtype = F64 if bits == 64 else F32
    p = O.params(dtype, K)
    for ktop in (0, 1, 2, FMT_KMAX[bits]):
        pool = EV.edge_pool(bits, K, ktop)
        # every value on its own, then random multisets
        sets = [[v] for v in pool] + [list(rng.choice(pool, int(rng.integers(2, 30)))) for _ in range(60)]
        for vals in sets:
            vals = [float(v) for v in vals]
            st = O.deposit_all(p, vals)
            ktop_cf, T = X.state_closed_form(vals, K, bits)
            S, C = X.canonical_SC(ktop_cf, T, bits)
            assert st.S == S and st.C == C, (vals, st, S, C)
            assert bits64(O.finalize(p, st)) == bits64(X.finalize_closed_form(ktop_cf, T, bits)), vals


FMT_KMAX = {64: 25, 32: 7}


@pytest.mark.parametrize("bits", [64, 32])
def test_edge_erange_limit(bits):
    # |b| >= 2^(W KMAX + W - 1 - m) needs a non-finite extractor (reading A-9)
    dtype = np.float64 if bits == 64 else np.float32
    lim = EV.erange_limit(bits)
    assert lim == (2.0 ** 987 if bits == 64 else 2.0 ** 120)
    k = np.zeros(3, np.int32)
    for K in (1, 2, 3):
        assert O.groupby_sum(k, np.array([1.0, lim, 2.0], dtype), 1, K)[0] == O.ERANGE
        assert O.groupby_sum(k, np.array([1.0, -lim, 2.0], dtype), 1, K)[0] == O.ERANGE
        rc, out = O.groupby_sum(k, np.array([0.0, EV.below(lim, bits), 0.0], dtype), 1, K)
        assert rc == O.OK
        if K >= 2:  # the value's bits span two levels: a single value round-trips
            assert float(out[0]) == EV.below(lim, bits)


def test_subnormals_and_signed_zero_give_positive_zero():
    # f = 0: subnormals lie below every ulp of the k = 0 window and contribute
    # nothing (reading A-11); zeros of either sign give +0.0
    for bits, dtype in ((64, np.float64), (32, np.float32)):
        vals = np.array(EV.subnormals(bits), dtype)
        for K in (1, 2, 3, 4):
            rc, out = O.groupby_sum(np.zeros(vals.size, np.int32), vals, 1, K)
            assert rc == O.OK and out.tobytes() == np.zeros(1, dtype).tobytes()


def test_half_unit_ties_round_away_from_zero():
    # (d + 1/2) u_1 at the top level of the k = 1 window: digit d + 1 (away
    # from zero) and remainder -u_1/2, i.e. digit -2^(W-1) at the next level
    # (reading A-1); hand-derived digits, then the oracle's state against them
    for bits, K in ((64, 2), (32, 2)):
        m, W, _ = EV.FMT[bits]
        dtype = F64 if bits == 64 else F32
        p = O.params(dtype, K)
        for d in (0, 1, 2, 7):
            for sgn in (1, -1):
                v = sgn * (d + 0.5) * 2.0 ** (W - m)
                T = [sgn * (d + 1), -sgn * (1 << (W - 1))]
                assert X.state_closed_form([v], K, bits) == (1, T)
                S, C = X.canonical_SC(1, T, bits)
                st = O.deposit_all(p, [v])
                assert st.S == S and st.C == C, (v, st, S, C)


# --------------------------------------------------------------------------
# binary32 carry counter limit (reading A-8): |C| >= 2^24 is ERANGE
# --------------------------------------------------------------------------

def test_f32_carry_limit_crafted_state():
    # canonical k = 0 state, D = 0: t_1 = 0.25 ufp C = C / 4 (exact for |C| < 2^24)
    p = O.params(F32, 2)
    for c in (2.0 ** 24, -(2.0 ** 24), 2.0 ** 24 + 2.0):
        with pytest.raises(ValueError, match=str(O.ERANGE)):
            O.finalize(p, O.State([1.5, 1.5 * 2.0 ** -18], [c, 0.0]))
    for c in (2.0 ** 24 - 1, -(2.0 ** 24 - 1), 12345.0):
        q = O.finalize(p, O.State([1.5, 1.5 * 2.0 ** -18], [c, 0.0]))
        assert q == float(np.float32(c / 4))


def test_f32_carry_limit_by_deposits():
    # b = the largest binary32 below 2^-6 has level-1 digit 2^17 at window 0:
    # n rows carry C_1 = n 2^17 / 2^21 = n / 16.  n = 2^28 reaches C = 2^24.
    b = np.float32(EV.below(2.0 ** -6, 32))
    assert float(b) == 2.0 ** -6 - 2.0 ** -30
    n = 1 << 28
    keys = np.zeros(n, np.int32)
    vals = np.full(n, b, np.float32)
    assert O.groupby_sum(keys, vals, 1, 2)[0] == O.ERANGE
    m = n - 16  # C = 2^24 - 1: readable; all value bits lie above ulp_2, so Q = RN(exact)
    rc, out = O.groupby_sum(keys[:m], vals[:m], 1, 2)
    exact = Fraction(m) * Fraction(float(b))
    assert rc == O.OK and float(out[0]) == X.round_to_binary(exact, 32) == 2.0 ** 22 - 0.5
