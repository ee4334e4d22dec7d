"""Oracle pins for the keyless single-array SUM and dot product (f4 of
SURVEY.md 8(f); the RSum setting): the closed form of
exact_ref.py (exact rationals, not the oracle's C code), products rounded
once by an exact-rational reference (reading A-19), exactness on integer
data, order invariance, and the degenerate cases."""
from fractions import Fraction

import numpy as np
import pytest

import exact_ref as X
import oracle as O


def _bits(x, dt):
    return np.asarray(x, dtype=dt).view(np.uint64 if dt == np.float64 else np.uint32).item()


def _values(rng, n, bits, spread):
    e = rng.integers(-spread, spread + 1, n)
    v = rng.uniform(1, 2, n) * np.exp2(e) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return v.astype(np.float64 if bits == 64 else np.float32)


@pytest.mark.parametrize("bits,K", [(64, 1), (64, 2), (64, 3), (64, 4), (32, 1), (32, 2), (32, 3), (32, 4)])
def test_rsum_equals_closed_form(bits, K):
    rng = np.random.default_rng(700 + bits + K)
    dt = np.float64 if bits == 64 else np.float32
    for _ in range(12):
        x = _values(rng, int(rng.integers(1, 200)), bits, 30 if bits == 64 else 12)
        rc, got = O.rsum(x, K, threads=1)
        assert rc == O.OK
        ktop, T = X.state_closed_form([float(v) for v in x], K, bits)
        assert _bits(got, dt) == _bits(X.finalize_closed_form(ktop, T, bits), dt)


@pytest.mark.parametrize("bits,K", [(64, 2), (64, 3), (32, 2), (32, 3)])
def test_dot_is_rsum_of_once_rounded_products(bits, K):
    """Each product is RN(x_i y_i) in the value type: derived here from
    exact rationals, independently of numpy's multiply."""
    rng = np.random.default_rng(800 + bits + K)
    dt = np.float64 if bits == 64 else np.float32
    for _ in range(8):
        n = int(rng.integers(1, 120))
        x, y = _values(rng, n, bits, 20 if bits == 64 else 8), _values(rng, n, bits, 20 if bits == 64 else 8)
        prods = [X.round_to_binary(Fraction(float(a)) * Fraction(float(b)), bits) for a, b in zip(x, y)]
        ktop, T = X.state_closed_form(prods, K, bits)
        rc, got = O.dot(x, y, K, threads=1)
        assert rc == O.OK
        assert _bits(got, dt) == _bits(X.finalize_closed_form(ktop, T, bits), dt)


def test_dot_exact_on_integer_data():
    rng = np.random.default_rng(9)
    x = rng.integers(-1000, 1000, 5000).astype(np.float64)
    y = rng.integers(-1000, 1000, 5000).astype(np.float64)
    rc, got = O.dot(x, y, 2)
    assert rc == O.OK
    assert got == float(sum(int(a) * int(b) for a, b in zip(x, y)))


def test_rsum_order_invariant_and_ones():
    rng = np.random.default_rng(10)
    x = _values(rng, 3000, 64, 40)
    ref = O.rsum(x, 3)[1]
    for _ in range(3):
        assert _bits(O.rsum(rng.permutation(x), 3)[1], np.float64) == _bits(ref, np.float64)
    # dot with a vector of ones deposits x itself
    assert _bits(O.dot(x, np.ones_like(x), 3)[1], np.float64) == _bits(ref, np.float64)


def test_rsum_degenerate_cases():
    rc, v = O.rsum(np.zeros(0, np.float64), 3)
    assert rc == O.OK and _bits(v, np.float64) == 0  # +0, not -0
    rc, v = O.rsum(np.array([-0.0, -0.0]), 3)
    assert rc == O.OK and _bits(v, np.float64) == 0
    rc, v = O.rsum(np.array([1.0, 2.0 ** 100, -(2.0 ** 100)]), 2)
    assert rc == O.OK and v == 0.0  # window top k*(2^100) = 3; K=2 keeps levels 3, 2 (unit 2^28): 1 rounds away
    rc, v = O.rsum(np.array([1.0, 2.0 ** 100, -(2.0 ** 100)]), 3)
    assert rc == O.OK and v == 1.0
    rc, _ = O.rsum(np.array([1.0, np.nan]), 3)
    assert rc == O.EDOM
    rc, _ = O.dot(np.array([np.inf, 1.0]), np.array([0.0, 1.0]), 3)  # inf * 0 = NaN
    assert rc == O.EDOM
