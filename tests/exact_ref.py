"""Exact-rational references used to pin the oracle (test infrastructure).

Nothing here calls or mirrors ``oracle/repro_oracle.c``: it is a second,
independent derivation of what the K-fold reproducible accumulator holds,
written with Python integers and ``fractions.Fraction`` only.

Closed form (derived from Alg. 1,
PAPER.md:654-687, under readings A-1..A-3):

* m, W = 52, 40 (binary64) or 23, 18 (binary32); f = 0.
* Absolute level j has unit u_j = 2^(W*j - m).  A value b needs the lattice
  index k*(b) = min{k >= 0 : |b| < 2^(W*k + W - 1 - m)} (Alg. 1 lines 3-9:
  |b| < 2^(W-1) ulp(S^(1))).  A group's window top is k_top = max k*(b).
* Digits: r = b; for j = k_top, k_top-1, ..., k_top-K+1:
  d_j = round-half-away(r / u_j); r -= d_j u_j     (Alg. 1 lines 10-16, A-1)
* T_j = sum of d_j over the group's rows (exact integers).
* Canonical state (Alg. 1 lines 17-21 keep S in [1.5, 1.75) ufp):
  D = T mod 2^(m-2), C = floor(T / 2^(m-2)), S = 1.5 * 2^(W*j) + D * u_j.
* Eq. 1: t_l = RN(D u + C 2^(W*j-2)); Q = t_K (+) ... (+) t_1.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

FMT = {64: (52, 40, 25), 32: (23, 18, 7)}  # m, W, largest lattice index


def round_half_away(x: Fraction) -> int:
    n, d = x.numerator, x.denominator  # d > 0
    q, r = divmod(abs(n), d)
    if 2 * r >= d:
        q += 1
    return q if n >= 0 else -q


def kstar(b: float, bits: int) -> int:
    m, W, _ = FMT[bits]
    a = abs(Fraction(b))
    k = 0
    while not (a < Fraction(2) ** (W * k + W - 1 - m)):
        k += 1
    return k


def round_to_binary(x: Fraction, bits: int) -> float:
    """Correctly rounded (nearest, ties to even) binary64/binary32 value of x."""
    if bits == 64:
        return float(x)  # CPython int/int true division is correctly rounded
    if x == 0:
        return 0.0
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    # a in [2^e, 2^(e+1)); binary32: 23 fraction bits, emin = -126, emax = 127
    q = max(e, -126) - 23
    scaled = a / Fraction(2) ** q
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    val = Fraction(n) * Fraction(2) ** q
    if val >= Fraction(2) ** 128 - Fraction(2) ** 103:  # round-to-nearest overflow
        return sign * math.inf
    return sign * float(val)


def fp_add(a: float, b: float, bits: int) -> float:
    if bits == 64:
        return a + b
    return float(np.float32(a) + np.float32(b))


def state_closed_form(values, K: int, bits: int):
    """(k_top, T[K]) of one group, T listed from the top level down."""
    m, W, _ = FMT[bits]
    ks = [kstar(b, bits) for b in values]
    ktop = max([0] + ks)
    T = [0] * K
    for b in values:
        r = Fraction(b)
        for l in range(K):
            j = ktop - l
            u = Fraction(2) ** (W * j - m)
            d = round_half_away(r / u)
            T[l] += d
            r -= d * u
    return ktop, T


def canonical_SC(ktop: int, T, bits: int):
    """Paper state <S, C> (floats, exact) of the closed-form integers."""
    m, W, _ = FMT[bits]
    S, C = [], []
    for l, t in enumerate(T):
        j = ktop - l
        D, Cl = t % (1 << (m - 2)), t // (1 << (m - 2))
        s = Fraction(3, 2) * Fraction(2) ** (W * j) + D * Fraction(2) ** (W * j - m)
        S.append(round_to_binary(s, bits))
        assert Fraction(S[-1]) == s  # exactly representable
        C.append(float(Cl))
    return S, C


def finalize_closed_form(ktop: int, T, bits: int) -> float:
    m, W, _ = FMT[bits]
    K = len(T)
    q = None
    for l in range(K - 1, -1, -1):
        j = ktop - l
        D, Cl = T[l] % (1 << (m - 2)), T[l] // (1 << (m - 2))
        t = round_to_binary(D * Fraction(2) ** (W * j - m) + Cl * Fraction(2) ** (W * j - 2), bits)
        q = t if q is None else fp_add(q, t, bits)
    return q


def represented_value(ktop: int, T, bits: int) -> Fraction:
    """V = sum_l T_l u_l: the exact value the (un-rounded) state represents."""
    m, W, _ = FMT[bits]
    return sum(Fraction(t) * Fraction(2) ** (W * (ktop - l) - m) for l, t in enumerate(T))


def exact_sum(values) -> Fraction:
    return sum((Fraction(v) for v in values), Fraction(0))


def lowest_ulp(ktop: int, K: int, bits: int) -> Fraction:
    m, W, _ = FMT[bits]
    return Fraction(2) ** (W * (ktop - K + 1) - m)
