"""Seeded synthetic inputs shaped like the paper's / BASELINE.json workloads.

This module holds NO arithmetic of the reproducible-sum method: it only
draws keys and values.  Both the CUDA path (tests, bench) and the CPU oracle
consume the same bytes from here.

Generator: counter-based SplitMix64 finaliser over (seed, column, row index),
so any shard or chunk of rows is reproducible on its own; range reduction by
multiply-shift ((h >> 32) * R) >> 32.  Seed = 0x1802098830 + config id.

Configs (BASELINE.json "configs"; the paper's own workload: n <key, value>
pairs with keys uniform in [0, n_groups)):
  0  2^16 rows, keys U[0,16),  fp64 +-(1 + mant52 2^-52) 2^e, e U{-20..20}, K=3
  1  2^27 rows, keys U[0,1024), values as config 0, K=3
  2  2^28 rows, keys U[0,G), G = 4^j, fp64 2 (h>>11) 2^-53 - 1 in [-1, 1), K=3
  3  2^28 rows, keys Zipf(s=1.1) over 2^20 groups, fp32 z 2^e with z a
     Box-Muller normal from two 53-bit uniforms, e U{-10..10}, K=2
  4  2^30 rows, keys U[0,4), qty 1+U{0..49}, price (90000+U{0..10410000})/100,
     disc U{0..10}/100, tax U{0..8}/100 (fp64), K=3
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x1802098830
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_COL = np.uint64(0xD6E8FEB86659FD93)

CONFIGS = {
    0: dict(n=1 << 16, n_groups=16, fold=3, dtype="f64", values="signed_mant_exp20"),
    1: dict(n=1 << 27, n_groups=1024, fold=3, dtype="f64", values="signed_mant_exp20"),
    2: dict(n=1 << 28, n_groups=None, fold=3, dtype="f64", values="uniform_pm1"),
    3: dict(n=1 << 28, n_groups=1 << 20, fold=2, dtype="f32", values="normal_exp10", keys="zipf1.1"),
    4: dict(n=1 << 30, n_groups=4, fold=3, dtype="f64", values="q1"),
}


def splitmix(seed: int, col: int, idx: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser of (seed, column, row index) -> uint64[len(idx)]."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(col) * _COL)
        z = z + (idx.astype(np.uint64) + np.uint64(1)) * _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_int(h: np.ndarray, R: int) -> np.ndarray:
    """Multiply-shift range reduction of the top 32 bits to [0, R), R < 2^32."""
    with np.errstate(over="ignore"):
        return ((h >> np.uint64(32)) * np.uint64(R)) >> np.uint64(32)


def _rows(r0: int, r1: int) -> np.ndarray:
    return np.arange(r0, r1, dtype=np.uint64)


def keys_uniform(seed: int, r0: int, r1: int, n_groups: int) -> np.ndarray:
    return uniform_int(splitmix(seed, 0, _rows(r0, r1)), n_groups).astype(np.int32)


def values_signed_mant_exp(seed: int, r0: int, r1: int, emax: int = 20) -> np.ndarray:
    """+-(1 + mant52 * 2^-52) * 2^e, e uniform in [-emax, emax], built from bits."""
    idx = _rows(r0, r1)
    h1 = splitmix(seed, 1, idx)
    h2 = splitmix(seed, 2, idx)
    mant = h1 & np.uint64((1 << 52) - 1)
    sign = h1 >> np.uint64(63)
    e = uniform_int(h2, 2 * emax + 1).astype(np.int64) - emax
    bits = (sign << np.uint64(63)) | ((e + 1023).astype(np.uint64) << np.uint64(52)) | mant
    return bits.view(np.float64)


def values_uniform_pm1(seed: int, r0: int, r1: int) -> np.ndarray:
    """2 * (h >> 11) * 2^-53 - 1 in [-1, 1) (exact)."""
    h = splitmix(seed, 1, _rows(r0, r1))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def values_normal_exp(seed: int, r0: int, r1: int, emax: int = 10) -> np.ndarray:
    """binary32(z * 2^e): z Box-Muller normal from two 53-bit uniforms."""
    idx = _rows(r0, r1)
    u1 = ((splitmix(seed, 1, idx) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53  # (0, 1]
    u2 = (splitmix(seed, 2, idx) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    e = uniform_int(splitmix(seed, 3, idx), 2 * emax + 1).astype(np.int64) - emax
    return np.ldexp(z, e).astype(np.float32)


def zipf_cdf(n_groups: int, s: float) -> np.ndarray:
    w = np.arange(1, n_groups + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def keys_zipf(seed: int, r0: int, r1: int, n_groups: int, s: float = 1.1, cdf=None) -> np.ndarray:
    """Zipf(s) ranks over n_groups by inverse CDF (binary search); key = rank - 1."""
    cdf = zipf_cdf(n_groups, s) if cdf is None else cdf
    u = (splitmix(seed, 0, _rows(r0, r1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.minimum(np.searchsorted(cdf, u, side="right"), n_groups - 1).astype(np.int32)


def keys_sparse(seed: int, r0: int, r1: int, distinct: int) -> np.ndarray:
    """Arbitrary int64 keys (the f1 workload): row id uniform in [0, distinct),
    key = SplitMix64 of the id (column 7) shifted to 62 bits -- `distinct`
    distinct keys spread over the int64 range, no order or density."""
    ids = uniform_int(splitmix(seed, 0, _rows(r0, r1)), distinct)
    return (splitmix(seed, 7, ids) >> np.uint64(2)).astype(np.int64)


def generate(config: int, n: int | None = None, n_groups: int | None = None, r0: int = 0,
             seed: int | None = None):
    """(keys int32[n], vals) for BASELINE config `config` (rows r0 .. r0+n)."""
    c = CONFIGS[config]
    n = c["n"] if n is None else n
    G = c["n_groups"] if n_groups is None else n_groups
    if G is None:
        raise ValueError("config 2 needs n_groups (a power of 4)")
    seed = SEED_BASE + config if seed is None else seed
    r1 = r0 + n
    if config in (0, 1):
        return keys_uniform(seed, r0, r1, G), values_signed_mant_exp(seed, r0, r1)
    if config == 2:
        return keys_uniform(seed, r0, r1, G), values_uniform_pm1(seed, r0, r1)
    if config == 3:
        return keys_zipf(seed, r0, r1, G), values_normal_exp(seed, r0, r1)
    if config == 4:
        idx = _rows(r0, r1)
        keys = keys_uniform(seed, r0, r1, G)
        qty = 1.0 + uniform_int(splitmix(seed, 1, idx), 50).astype(np.float64)
        price = (90000.0 + uniform_int(splitmix(seed, 2, idx), 10410001).astype(np.float64)) / 100.0
        disc = uniform_int(splitmix(seed, 3, idx), 11).astype(np.float64) / 100.0
        tax = uniform_int(splitmix(seed, 4, idx), 9).astype(np.float64) / 100.0
        return keys, (qty, price, disc, tax)
    raise ValueError(config)


def generate_chunked(config: int, n: int, n_groups: int | None, chunk: int = 1 << 24):
    """Generate in chunks (bounded temporaries); returns the concatenated arrays."""
    c = CONFIGS[config]
    vt = np.float32 if c["dtype"] == "f32" else np.float64
    keys = np.empty(n, dtype=np.int32)
    vals = np.empty(n, dtype=vt)
    cdf = zipf_cdf(n_groups, 1.1) if config == 3 else None
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        if config == 3:
            seed = SEED_BASE + 3
            keys[r0:r1] = keys_zipf(seed, r0, r1, n_groups, cdf=cdf)
            vals[r0:r1] = values_normal_exp(seed, r0, r1)
        else:
            k, v = generate(config, n=r1 - r0, n_groups=n_groups, r0=r0)
            keys[r0:r1] = k
            vals[r0:r1] = v
    return keys, vals
