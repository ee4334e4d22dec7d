"""Edge-case values of the K-fold accumulator's domain (test inputs only).

Built from the lattice constants of DESIGN.md section 2 (m, W per format,
f = 0): the window-top thresholds 2^(W k + W - 1 - m) of Alg. 1 line 3
 and the values just below them, subnormals and signed zeros
(reading A-11), and half-unit ties (d + 1/2) u_l at every level of a window
(reading A-1: the extraction q = (r (+) S) (-) S rounds them away from
zero).  Nothing here computes a digit or a sum.
"""
from __future__ import annotations

import numpy as np

# m, W, largest lattice index (reading A-9)
FMT = {64: (52, 40, 25), 32: (23, 18, 7)}


def np_type(bits):
    return np.float64 if bits == 64 else np.float32


def exact(x, bits):
    """x is a value of the format (numpy 2 compares a float32 with a Python
    float in float32, so compare as Python floats)."""
    return float(np_type(bits)(x)) == float(x)


def below(x, bits):
    t = np_type(bits)
    return float(np.nextafter(t(x), t(0)))


def threshold(k, bits):
    """Smallest |b| that needs a window top above k."""
    m, W, _ = FMT[bits]
    return 2.0 ** (W * k + W - 1 - m)


def erange_limit(bits):
    """|b| >= this is ERANGE (the top extractor 1.5 * 2^(W (KMAX + 1)) overflows)."""
    return threshold(FMT[bits][2], bits)


def thresholds(bits):
    """At and just below every threshold that keeps k* <= KMAX, both signs."""
    _, _, kmax = FMT[bits]
    out = []
    for k in range(kmax + 1):
        t = threshold(k, bits)
        if k < kmax:
            out += [t, -t]
        out += [below(t, bits), -below(t, bits)]
    return out


def subnormals(bits):
    t = np_type(bits)
    fi = np.finfo(t)
    tiny = float(fi.smallest_subnormal)
    top = float(np.nextafter(t(fi.tiny), t(0)))  # largest subnormal
    mid = float(t(tiny * 12345))
    return [tiny, -tiny, top, -top, mid, -mid, 0.0, -0.0]


def ties(bits, K, ktop):
    """(d + 1/2) u_l at each level l of the window with top ktop, both signs,
    and compound values a u_0 + (d + 1/2) u_l; all below threshold(ktop)."""
    m, W, _ = FMT[bits]
    out = []
    for l in range(K):
        u = 2.0 ** (W * (ktop - l) - m)
        for d in (0, 1, 2, 3, 7, 12345):
            v = (d + 0.5) * u
            if abs(v) < threshold(ktop, bits) and v != 0.0:
                out += [v, -v]
        if l > 0:
            u0 = 2.0 ** (W * ktop - m)
            for a, d in ((1, 0), (3, 5), (5, 2)):
                v = a * u0 + (d + 0.5) * u
                if exact(v, bits) and abs(v) < threshold(ktop, bits):
                    out += [v, -v, a * u0 - (d + 0.5) * u]
    return [x for x in out if exact(x, bits)]


def anchor(bits, ktop):
    """A value whose window top is exactly ktop (k* = ktop)."""
    return 0.75 * threshold(ktop, bits) if ktop > 0 else 0.5 * threshold(0, bits)


def edge_pool(bits, K, ktop):
    """Every edge value that keeps a group's window top <= ktop, except that
    the thresholds above ktop are included too (they raise the top)."""
    return thresholds(bits) + subnormals(bits) + ties(bits, K, ktop) + [anchor(bits, ktop)]


def edge_rows(rng, bits, K, G, n, ktops=(0, 1, 2)):
    """n rows over G groups: each group draws mostly from the ties and
    subnormals of one window (ktop cycled over `ktops`, anchored by one value
    at that window), plus threshold values spread over every group and a
    normal background.  Returns (keys int32[n], vals)."""
    t = np_type(bits)
    keys = rng.integers(0, G, n).astype(np.int32)
    vals = np.empty(n, dtype=t)
    thr = np.array(thresholds(bits), dtype=t)
    sub = np.array(subnormals(bits), dtype=t)
    pools = {k: np.array(ties(bits, K, k) + [anchor(bits, k)], dtype=t) for k in ktops}
    kt = np.array(ktops)[np.arange(G) % len(ktops)]
    u = rng.random(n)
    for i in range(n):
        g = keys[i]
        if u[i] < 0.02:
            vals[i] = thr[rng.integers(0, thr.size)]
        elif u[i] < 0.10:
            vals[i] = sub[rng.integers(0, sub.size)]
        elif u[i] < 0.75:
            p = pools[int(kt[g])]
            vals[i] = p[rng.integers(0, p.size)]
        else:
            vals[i] = t(rng.standard_normal() * threshold(int(kt[g]), bits) / 4)
    return keys, vals
