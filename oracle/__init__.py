"""CPU oracle for the reproducible GroupBy-SUM of arxiv 1802.09883.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
package.  It loads ``oracle/liboracle.so`` (built from ``repro_oracle.c`` by
:func:`build`), which shares no code with the CUDA path.

Every function maps one-to-one onto a C function of ``repro_oracle.c``; the
paper passages each one follows are cited there (Alg. 1 PAPER.md:654-687,
Eq. 1, merge SPEC.md:186-195, GroupBy PAPER.md:291-302).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "repro_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EKEY, EDOM, ERANGE, ENOMEM = 0, -1, -2, -3, -4, -6
KIND_F64, KIND_F32, KIND_TOY = 0, 1, 2
F32, F64 = 0, 1  # dtype codes (same numbering as the C-ABI, defined separately)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -ffp-contract=off (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class Params(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("m", ctypes.c_int), ("W", ctypes.c_int),
                ("f", ctypes.c_int), ("L", ctypes.c_int), ("emin", ctypes.c_int),
                ("emax", ctypes.c_int), ("ties_away", ctypes.c_int),
                ("thr_shift", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, P, dp = ctypes.c_double, ctypes.POINTER(Params), ctypes.POINTER(ctypes.c_double)
        L.orc_ufp.argtypes, L.orc_ufp.restype = [d], d
        L.orc_ulp.argtypes, L.orc_ulp.restype = [P, d], d
        L.orc_lsb_force.argtypes, L.orc_lsb_force.restype = [P, d], d
        L.orc_eft.argtypes, L.orc_eft.restype = [P, d, d, dp, dp], None
        L.orc_fadd.argtypes, L.orc_fadd.restype = [P, d, d], d
        L.orc_round.argtypes, L.orc_round.restype = [P, d], d
        L.orc_init.argtypes, L.orc_init.restype = [P, dp, dp], ctypes.c_int
        L.orc_deposit.argtypes, L.orc_deposit.restype = [P, dp, dp, d], ctypes.c_int
        L.orc_merge.argtypes, L.orc_merge.restype = [P, dp, dp, dp, dp], ctypes.c_int
        L.orc_finalize.argtypes, L.orc_finalize.restype = [P, dp, dp, dp], ctypes.c_int
        L.orc_carry.argtypes, L.orc_carry.restype = [P, dp, dp], None
        L.orc_params_for.argtypes, L.orc_params_for.restype = [P, ctypes.c_int, ctypes.c_int], ctypes.c_int
        vp = ctypes.c_void_p
        L.orc_groupby_sum.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, vp, vp, ctypes.c_int, ctypes.c_int]
        L.orc_groupby_sum.restype = ctypes.c_int
        L.orc_groupby_sum_select.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_int32, vp, ctypes.c_int32, vp, vp, ctypes.c_int]
        L.orc_groupby_sum_select.restype = ctypes.c_int
        L.orc_plain_sum.argtypes, L.orc_plain_sum.restype = [P, vp, ctypes.c_int64], d
        _lib = L
    return _lib


def params(dtype: int | None = None, K: int = 3, *, m: int | None = None, W: int | None = None,
           f: int = 0, emin: int = -1022, emax: int = 1023, ties_away: bool = True,
           thr_shift: int | None = None) -> Params:
    """Production parameters (dtype given) or a toy format (m, W given)."""
    p = Params()
    if dtype is not None:
        st = lib().orc_params_for(ctypes.byref(p), dtype, K)
        assert st == OK
    else:
        p.kind, p.m, p.W, p.L, p.emin, p.emax = KIND_TOY, m, W, K, emin, emax
    p.f = f if dtype is None else p.f
    p.ties_away = 1 if ties_away else 0
    p.thr_shift = (p.W - 1) if thr_shift is None else thr_shift
    return p


@dataclass
class State:
    """<S, C> of one reproducible accumulator."""
    S: list
    C: list

    def key(self):
        return tuple(np.float64(x).view(np.uint64).item() for x in self.S + self.C)


def _arr(vals):
    return (ctypes.c_double * len(vals))(*vals)


def init(p: Params) -> State:
    S, C = (ctypes.c_double * p.L)(), (ctypes.c_double * p.L)()
    assert lib().orc_init(ctypes.byref(p), S, C) == OK
    return State(list(S), list(C))


def deposit(p: Params, st: State, b: float) -> int:
    S, C = _arr(st.S), _arr(st.C)
    rc = lib().orc_deposit(ctypes.byref(p), S, C, float(b))
    st.S, st.C = list(S), list(C)
    return rc


def deposit_all(p: Params, values, st: State | None = None) -> State:
    st = init(p) if st is None else st
    for b in values:
        rc = deposit(p, st, b)
        if rc != OK:
            raise ValueError(f"deposit failed: {rc}")
    return st


def merge(p: Params, dst: State, src: State) -> int:
    S, C = _arr(dst.S), _arr(dst.C)
    rc = lib().orc_merge(ctypes.byref(p), S, C, _arr(src.S), _arr(src.C))
    dst.S, dst.C = list(S), list(C)
    return rc


def finalize(p: Params, st: State) -> float:
    q = ctypes.c_double()
    rc = lib().orc_finalize(ctypes.byref(p), _arr(st.S), _arr(st.C), ctypes.byref(q))
    if rc != OK:
        raise ValueError(f"finalize failed: {rc}")
    return q.value


def carry(p: Params, S: float, C: float):
    s, c = ctypes.c_double(S), ctypes.c_double(C)
    lib().orc_carry(ctypes.byref(p), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def eft(p: Params, a: float, b: float):
    q, r = ctypes.c_double(), ctypes.c_double()
    lib().orc_eft(ctypes.byref(p), a, b, ctypes.byref(q), ctypes.byref(r))
    return q.value, r.value


def ufp(x: float) -> float:
    return lib().orc_ufp(x)


def ulp(p: Params, x: float) -> float:
    return lib().orc_ulp(ctypes.byref(p), x)


def lsb_force(p: Params, x: float) -> float:
    return lib().orc_lsb_force(ctypes.byref(p), x)


def fadd(p: Params, a: float, b: float) -> float:
    return lib().orc_fadd(ctypes.byref(p), a, b)


def fround(p: Params, x: float) -> float:
    return lib().orc_round(ctypes.byref(p), x)


def plain_sum(p: Params, values) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().orc_plain_sum(ctypes.byref(p), v.ctypes.data, v.size)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def groupby_sum(keys: np.ndarray, vals: np.ndarray, n_groups: int, fold: int, *,
                threads: int | None = None, mode: int = 0, with_state: bool = False):
    """GroupBy-SUM (O5/O6).  Returns (status, out[, state]); state is
    [n_groups, 2K] float64 rows S[0..K) then C[0..K) (SPEC.md:277 layout)."""
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    dtype = F64 if vals.dtype == np.float64 else F32
    vals = np.ascontiguousarray(vals)
    assert vals.dtype in (np.float64, np.float32)
    out = np.zeros(n_groups, dtype=vals.dtype)
    state = np.zeros((n_groups, 2 * fold), dtype=np.float64) if with_state else None
    rc = lib().orc_groupby_sum(keys.ctypes.data, vals.ctypes.data, keys.size, n_groups, fold,
                               dtype, out.ctypes.data,
                               state.ctypes.data if with_state else None,
                               threads or default_threads(), mode)
    return (rc, out, state) if with_state else (rc, out)


def groupby_sum_select(keys: np.ndarray, vals: np.ndarray, n_groups: int, fold: int,
                       sel: np.ndarray, *, threads: int | None = None, with_state: bool = False):
    """GroupBy-SUM restricted to the groups in ``sel`` (outputs indexed like sel)."""
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    dtype = F64 if vals.dtype == np.float64 else F32
    vals = np.ascontiguousarray(vals)
    out = np.zeros(sel.size, dtype=vals.dtype)
    state = np.zeros((sel.size, 2 * fold), dtype=np.float64) if with_state else None
    rc = lib().orc_groupby_sum_select(keys.ctypes.data, vals.ctypes.data, keys.size, n_groups,
                                      fold, dtype, sel.ctypes.data, sel.size, out.ctypes.data,
                                      state.ctypes.data if with_state else None,
                                      threads or default_threads())
    return (rc, out, state) if with_state else (rc, out)


_PRECEDENCE = (EKEY, EDOM, ERANGE)


def q1_project(price: np.ndarray, disc: np.ndarray, tax: np.ndarray):
    """Config-4 row projection, reading A-15: disc_price =
    price (x) (1 (-) disc), charge = disc_price (x) (1 (+) tax), each
    operation one binary64 rounding (numpy elementwise ops, no contraction)."""
    one = np.float64(1.0)
    disc_price = np.multiply(price, np.subtract(one, disc))
    charge = np.multiply(disc_price, np.add(one, tax))
    return disc_price, charge


def groupby_sum_multi(keys: np.ndarray, cols, n_groups: int, fold: int, proj: int = 0, *,
                      threads: int | None = None):
    """Several GroupBy-SUMs of one key column plus COUNT (the C-ABI's
    repro_groupby_sum_multi): each output column is O5 on its value column
    (proj 1: on the projected columns of q1_project); COUNT is the number of
    rows per group.  Status: the highest-precedence error of any column
    (EKEY > EDOM > ERANGE).  Returns (status, [outs], counts)."""
    keys = np.ascontiguousarray(keys, dtype=np.int32)
    if proj == 1:
        qty, price, disc, tax = cols
        dp, ch = q1_project(price, disc, tax)
        cols = [qty, price, dp, ch]
    elif proj == 2:
        x = np.ascontiguousarray(cols[0])
        cols = [x, np.multiply(x, x)]  # one rounding per square
    outs, codes = [], []
    for c in cols:
        rc, o = groupby_sum(keys, np.ascontiguousarray(c), n_groups, fold, threads=threads)
        outs.append(o)
        codes.append(rc)
    status = next((e for e in _PRECEDENCE if e in codes), OK)
    ok = (keys >= 0) & (keys < n_groups)
    counts = np.bincount(keys[ok], minlength=n_groups).astype(np.int64)
    return status, outs, counts


def groupby_moments(keys: np.ndarray, vals: np.ndarray, n_groups: int, fold: int, *, threads: int | None = None):
    """Per-group SUM, AVG, sample VARIANCE, STDDEV, COUNT from the reproducible
    SUM(x), SUM(x*x) and COUNT (groupby_sum_multi proj 2), with the formulas
    of repro_groupby_moments evaluated in the value type, one rounding per
    operation in the documented order (numpy elementwise ops)."""
    rc, (s, q), c = groupby_sum_multi(keys, [vals], n_groups, fold, proj=2, threads=threads)
    dt = vals.dtype.type
    cf = c.astype(vals.dtype)
    one, zero = dt(1), dt(0)
    with np.errstate(divide="ignore", invalid="ignore"):
        avg = np.where(c > 0, np.divide(s, cf), zero).astype(vals.dtype)
        t = np.subtract(q, np.divide(np.multiply(s, s), cf))
        var = np.where(c > 1, np.maximum(zero, np.divide(t, np.subtract(cf, one))), zero).astype(vals.dtype)
    sd = np.sqrt(var).astype(vals.dtype)
    return rc, {"sum": s, "avg": avg, "var": var, "stddev": sd, "count": c}


def rsum(x: np.ndarray, fold: int, *, threads: int | None = None):
    """Reproducible SUM of one array -- the RSum setting:
    one accumulator over every element (O5 with the single group 0).
    Returns (status, value)."""
    x = np.ascontiguousarray(x)
    rc, out = groupby_sum(np.zeros(x.size, np.int32), x, 1, fold, threads=threads)
    return rc, out[0]


def dot(x: np.ndarray, y: np.ndarray, fold: int, *, threads: int | None = None):
    """Reproducible dot product: each product x_i * y_i rounded once in the
    value type (numpy elementwise multiply, reading A-19), then rsum.
    Returns (status, value)."""
    x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
    assert x.dtype == y.dtype and x.size == y.size
    with np.errstate(invalid="ignore", over="ignore"):
        prod = np.multiply(x, y)
    return rsum(prod, fold, threads=threads)


INT64_MIN = np.iinfo(np.int64).min


def groupby_sum_sparse(keys: np.ndarray, vals: np.ndarray, fold: int, *, threads: int | None = None):
    """GroupBy-SUM over arbitrary int64 keys (the C-ABI's
    repro_groupby_sum_sparse): the distinct keys ascending (np.unique) and O5
    on the dense ids = rank of each row's key.  INT64_MIN is reserved (EKEY).
    Returns (status, distinct keys, sums)."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    if np.any(keys == INT64_MIN):
        return EKEY, np.zeros(0, np.int64), np.zeros(0, vals.dtype)
    uniq = np.unique(keys)
    if uniq.size == 0:
        return OK, uniq, np.zeros(0, vals.dtype)
    ids = np.searchsorted(uniq, keys).astype(np.int32)
    rc, out = groupby_sum(ids, vals, int(uniq.size), fold, threads=threads)
    return rc, uniq, out
