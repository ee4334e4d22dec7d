"""B200-native reproducible GroupBy-SUM (arxiv 1802.09883).

Thin ctypes binding over the C-ABI of ``include/repro_groupby.h``
(``_lib/librepro_b200.so``, hand-written sm_100a kernels).  Every function
here only marshals arguments: torch tensors are passed as device pointers and
every step of the GroupBy runs in the library's kernels.  There is no CPU
fallback: importing the package fails loudly when the library is missing.

Entry points mirror the C names:
  groupby_sum / groupby_sum_async / groupby_sum_host / workspace_bytes
  groupby_sum_multi / groupby_sum_multi_async / multi_workspace_bytes
  Accumulator (repro_acc_*), baseline_atomic_sum, and introspection helpers.
"""
from __future__ import annotations

import ctypes
import os

from .build_native import LIB as _LIB_PATH

F32, F64 = 0, 1
OK, EINVAL, EKEY, EDOM, ERANGE, ECUDA, ENOMEM = 0, -1, -2, -3, -4, -5, -6
_STATUS = {0: "OK", -1: "EINVAL", -2: "EKEY", -3: "EDOM", -4: "ERANGE", -5: "ECUDA", -6: "ENOMEM"}

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"librepro_b200.so not found at {_LIB_PATH}: build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

_lib = ctypes.CDLL(_LIB_PATH)
LIB_PATH = _LIB_PATH

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("repro_strerror", ctypes.c_char_p, ctypes.c_int)
_sig("repro_version", ctypes.c_char_p)
_sig("repro_groupby_sum", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp)
_sig("repro_groupby_workspace_bytes", _sz, _i64, _i32, _i32, _i32)
_sig("repro_groupby_sum_async", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _vp, _vp)
_sig("repro_groupby_sum_host", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp)
_sig("repro_groupby_table", ctypes.c_int, _i64, _i32, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64))
_sig("repro_nvls_table_allreduce_async", ctypes.c_int, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _i32, _i32, _vp)
_sig("repro_groupby_deposit_async", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _sz, _vp)
_sig("repro_groupby_finish_async", ctypes.c_int, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _vp, _vp)
_sig("repro_groupby_window_limbs_async", ctypes.c_int, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _vp)
_sig("repro_groupby_finish_limbs_async", ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz,
     _vp, _vp)
_sig("repro_release_cache", None)
_sig("repro_synth_generate", ctypes.c_int, _i32, ctypes.c_uint64, _i64, _i64, _i32, _vp, ctypes.POINTER(_vp), _vp)
_sig("repro_groupby_sum_multi", ctypes.c_int, _vp, ctypes.POINTER(_vp), _i32, _i32, _i64, _i32, _i32, _i32,
     ctypes.POINTER(_vp), _vp)
_sig("repro_groupby_multi_workspace_bytes", _sz, _i64, _i32, _i32, _i32, _i32, _i32)
_sig("repro_groupby_sum_sparse", ctypes.c_int, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp, ctypes.POINTER(_i64))
_sig("repro_groupby_sum_sparse_i32", ctypes.c_int, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp, ctypes.POINTER(_i64))
_sig("repro_groupby_moments", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp)
_sig("repro_groupby_multi_table", ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_i64),
     ctypes.POINTER(_i64))
_sig("repro_groupby_multi_deposit_async", ctypes.c_int, _vp, ctypes.POINTER(_vp), _i32, _i32, _i64, _i32, _i32, _i32,
     _vp, _sz, _vp)
_sig("repro_groupby_multi_finish_async", ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp), _vp,
     _vp, _sz, _vp, _vp)
_sig("repro_groupby_sum_multi_async", ctypes.c_int, _vp, ctypes.POINTER(_vp), _i32, _i32, _i64, _i32, _i32, _i32,
     ctypes.POINTER(_vp), _vp, _vp, _sz, _vp, _vp)
_sig("repro_sum", ctypes.c_int, _vp, _i64, _i32, _i32, _vp)
_sig("repro_dot", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _vp)
_sig("repro_dot_workspace_bytes", _sz, _i32, _i32)
_sig("repro_dot_async", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _sz, _vp, _vp)
_sig("repro_dot_table", ctypes.c_int, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64))
_sig("repro_dot_deposit_async", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _vp, _sz, _vp)
_sig("repro_dot_finish_async", ctypes.c_int, _i32, _i32, _vp, _vp, _sz, _vp, _vp)
_sig("repro_tune_get", ctypes.c_int, _i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32))
_sig("repro_tune_set", ctypes.c_int, _i32, _i32, _i32, _i32)
_sig("repro_autotune", ctypes.c_int, _i64, _i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32))
_sig("repro_acc_create", ctypes.c_int, ctypes.POINTER(_vp), _i32, _i32, _i32)
_sig("repro_acc_deposit", ctypes.c_int, _vp, _vp, _vp, _i64)
_sig("repro_acc_merge", ctypes.c_int, _vp, _vp)
_sig("repro_acc_finalize", ctypes.c_int, _vp, _vp)
_sig("repro_acc_export", ctypes.c_int, _vp, _vp)
_sig("repro_acc_import", ctypes.c_int, _vp, _vp)
_sig("repro_acc_reset", ctypes.c_int, _vp)
_sig("repro_acc_destroy", None, _vp)
_sig("repro_acc_n_groups", _i32, _vp)
_sig("repro_acc_fold", _i32, _vp)
_sig("repro_acc_dtype", _i32, _vp)
_sig("repro_acc_top_levels", ctypes.c_int, _vp, _vp)
_sig("repro_acc_window_export", ctypes.c_int, _vp, _vp, _vp)
_sig("repro_acc_window_import", ctypes.c_int, _vp, _vp, _vp)
_sig("repro_acc_window_import_range", ctypes.c_int, _vp, _i32, _i32, _vp, _vp)
_sig("repro_baseline_atomic_sum", ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp)
_sig("repro_measure_fp_add_rate", ctypes.c_int, _i32, ctypes.POINTER(ctypes.c_double), _vp)
_sig("repro_last_launch_count", _i32)
_sig("repro_last_path", _i32)
_sig("repro_onchip_max_groups", _i32, _i32, _i32)
_sig("repro_sweep_max_groups", _i32, _i32, _i32)
_sig("repro_set_path_override", None, _i32)
_sig("repro_set_kernel_variant", None, _i32)
_sig("repro_set_route_mode", None, _i32)
_sig("repro_timing_enable", None, _i32)
_sig("repro_timing_collect", _i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_i32),
     ctypes.POINTER(ctypes.c_double), _i32)


class ReproError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = _lib.repro_strerror(status).decode()
        super().__init__(f"{what}: {_STATUS.get(status, status)} ({msg})")


def _check(status: int, what: str):
    if status != OK:
        raise ReproError(status, what)


def version() -> str:
    return _lib.repro_version().decode()


def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"values must be float32 or float64, got {t.dtype}")


def _dev(t, name, dtype=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.data_ptr() if t.numel() else None


def _need(t, n: int, name: str):
    """The C-ABI cannot see buffer sizes: check them here (ValueError, not a
    device out-of-bounds access)."""
    if t is not None and t.numel() < n:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {n}")


def _same_len(a, b, what: str = "keys and vals"):
    if a.numel() != b.numel():
        raise ValueError(f"{what} differ in length")


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def groupby_sum(keys, vals, n_groups: int, fold: int = 3, out=None):
    """Reproducible GroupBy-SUM (blocking).  keys int32[n], vals f32/f64[n] on CUDA."""
    torch = _torch()
    dt = _dtype_code(vals)
    _same_len(keys, vals)
    if out is None:
        out = torch.empty(n_groups, dtype=vals.dtype, device=vals.device)
    _need(out, n_groups, "out")
    st = _lib.repro_groupby_sum(_dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel(),
                                n_groups, fold, dt, _dev(out, "out", vals.dtype))
    _check(st, "repro_groupby_sum")
    return out


def workspace_bytes(n: int, n_groups: int, fold: int, dtype: int) -> int:
    return _lib.repro_groupby_workspace_bytes(n, n_groups, fold, dtype)


def make_workspace(n: int, n_groups: int, fold: int, dtype: int, device="cuda"):
    torch = _torch()
    nbytes = workspace_bytes(n, n_groups, fold, dtype)
    if nbytes == 0:
        raise ReproError(EINVAL, "repro_groupby_workspace_bytes")
    return torch.empty(nbytes + 256, dtype=torch.uint8, device=device)


def _aligned_ptr(ws):
    p = ws.data_ptr()
    return (p + 255) // 256 * 256, ws.numel() - ((p + 255) // 256 * 256 - p)


def groupby_sum_async(keys, vals, n_groups: int, fold: int, out, workspace, status, stream=None):
    """Enqueue the GroupBy on `stream` (default: current) with a caller
    workspace (make_workspace) and an int32 device status word."""
    torch = _torch()
    dt = _dtype_code(vals)
    _same_len(keys, vals)
    _need(out, n_groups, "out")
    _need(status, 1, "status")
    wp, wb = _aligned_ptr(workspace)
    st = _lib.repro_groupby_sum_async(_dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel(), n_groups,
                                      fold, dt, _dev(out, "out", vals.dtype), wp, wb, _stream_ptr(stream),
                                      _dev(status, "status", torch.int32))
    _check(st, "repro_groupby_sum_async")


# ---- split form of the single-column GroupBy (multi-GPU exchange) --------------

def groupby_table_views(workspace, n: int, n_groups: int, fold: int, dtype: int):
    """(flags int32[1], kglob int32[G], slots int64[G * NS * 2]) views of the
    absolute-level slot table a groupby_deposit_async leaves in `workspace`."""
    torch = _torch()
    off, cnt = (_i64 * 3)(), (_i64 * 3)()
    _check(_lib.repro_groupby_table(n, n_groups, fold, dtype, off, cnt), "repro_groupby_table")
    base = _aligned_ptr(workspace)[0] - workspace.data_ptr()
    return tuple(workspace[base + o: base + o + c * sz].view(dt)
                 for o, c, dt, sz in zip(off, cnt, (torch.int32, torch.int32, torch.int64), (4, 4, 8)))


def table_layout(n: int, n_groups: int, fold: int, dtype: int):
    """(offsets, counts) of the status word / kglob / slots regions of the
    single-column slot table (bytes from the aligned workspace start)."""
    off, cnt = (_i64 * 3)(), (_i64 * 3)()
    _check(_lib.repro_groupby_table(n, n_groups, fold, dtype, off, cnt), "repro_groupby_table")
    return list(off), list(cnt)


def nvls_table_allreduce_async(mc_workspace: int, offsets, counts, rank: int, world: int, stream=None):
    """In-switch all-reduce of a slot table through the multicast address of
    the aligned workspace (repro_nvls_table_allreduce_async)."""
    off, cnt = (_i64 * 3)(*offsets), (_i64 * 3)(*counts)
    _check(_lib.repro_nvls_table_allreduce_async(mc_workspace, off, cnt, rank, world, _stream_ptr(stream)),
           "repro_nvls_table_allreduce_async")


def groupby_deposit_async(keys, vals, n_groups: int, fold: int, workspace, stream=None):
    """Zero the workspace's slot table and deposit these rows into it."""
    torch = _torch()
    dt = _dtype_code(vals)
    _same_len(keys, vals)
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_groupby_deposit_async(_dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel(),
                                            n_groups, fold, dt, wp, wb, _stream_ptr(stream)),
           "repro_groupby_deposit_async")


def groupby_finish_async(n: int, n_groups: int, fold: int, dtype: int, out, workspace, status, stream=None):
    """Eq. 1 read-out of every group from the (all-reduced) slot table."""
    torch = _torch()
    _need(out, n_groups, "out")
    _need(status, 1, "status")
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_groupby_finish_async(n, n_groups, fold, dtype, _dev(out, "out"), wp, wb, _stream_ptr(stream),
                                           _dev(status, "status", torch.int32)), "repro_groupby_finish_async")
    return out


def groupby_window_limbs_async(n: int, n_groups: int, fold: int, dtype: int, k_global, limbs, workspace,
                               stream=None):
    """limbs int64[G * fold * 2] <- the slot words under the global tops."""
    torch = _torch()
    _need(k_global, n_groups, "k_global")
    _need(limbs, n_groups * fold * 2, "limbs")
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_groupby_window_limbs_async(n, n_groups, fold, dtype, _dev(k_global, "k_global", torch.int32),
                                                 _dev(limbs, "limbs", torch.int64), wp, wb, _stream_ptr(stream)),
           "repro_groupby_window_limbs_async")
    return limbs


def groupby_finish_limbs_async(n: int, n_groups: int, fold: int, dtype: int, g0: int, count: int, k_range,
                               limbs_range, out_range, workspace, status, stream=None):
    """Eq. 1 read-out of groups [g0, g0 + count) from summed limbs."""
    torch = _torch()
    if count:
        _need(k_range, count, "k_range")
        _need(limbs_range, count * fold * 2, "limbs_range")
        _need(out_range, count, "out_range")
    _need(status, 1, "status")
    wp, wb = _aligned_ptr(workspace)
    ptr = (lambda t, name, dt=None: _dev(t, name, dt) if count else None)
    _check(_lib.repro_groupby_finish_limbs_async(n, n_groups, fold, dtype, g0, count,
                                                 ptr(k_range, "k_range", torch.int32),
                                                 ptr(limbs_range, "limbs_range", torch.int64),
                                                 ptr(out_range, "out_range"), wp, wb, _stream_ptr(stream),
                                                 _dev(status, "status", torch.int32)),
           "repro_groupby_finish_limbs_async")


def groupby_sum_host(keys, vals, n_groups: int, fold: int = 3, out=None):
    """GroupBy from HOST (CPU, ideally pinned) tensors; returns a CPU tensor."""
    torch = _torch()
    if keys.is_cuda or vals.is_cuda:
        raise TypeError("groupby_sum_host takes host tensors")
    keys = keys.contiguous()
    vals = vals.contiguous()
    if keys.dtype != torch.int32:
        raise TypeError("keys must be int32")
    dt = _dtype_code(vals)
    _same_len(keys, vals)
    if out is None:
        out = torch.empty(n_groups, dtype=vals.dtype)
    _need(out, n_groups, "out")
    if out.is_cuda or out.dtype != vals.dtype or not out.is_contiguous():
        raise TypeError("out must be a contiguous host tensor of the value dtype")
    st = _lib.repro_groupby_sum_host(keys.data_ptr() if keys.numel() else None,
                                     vals.data_ptr() if vals.numel() else None, keys.numel(), n_groups, fold,
                                     dt, out.data_ptr())
    _check(st, "repro_groupby_sum_host")
    return out


def _multi_args(keys, cols, n_groups, proj, outs, counts):
    torch = _torch()
    if not cols:
        raise ValueError("at least one value column")
    dt = _dtype_code(cols[0])
    n = keys.numel()
    for c in cols:
        if c.dtype != cols[0].dtype or c.numel() != n:
            raise ValueError("value columns must share dtype and length with keys")
    nout = 4 if proj == 1 else 2 if proj == 2 else len(cols)
    if outs is None:
        outs = [torch.empty(n_groups, dtype=cols[0].dtype, device=cols[0].device) for _ in range(nout)]
    if len(outs) < nout:
        raise ValueError(f"{nout} output columns needed, got {len(outs)}")
    for o in outs:
        _need(o, n_groups, "outs[i]")
    _need(counts, n_groups, "counts")
    cptr = (_vp * len(cols))(*[_dev(c, "cols") for c in cols])
    optr = (_vp * len(outs))(*[_dev(o, "outs", cols[0].dtype) for o in outs])
    cnt = _dev(counts, "counts", torch.int64) if counts is not None else None
    return dt, n, outs, cptr, optr, cnt


def groupby_sum_multi(keys, cols, n_groups: int, fold: int = 3, proj: int = 0, outs=None, counts=None,
                      with_counts: bool = True):
    """Several reproducible SUMs (+ COUNT) of one key column in one pass
    (repro_groupby_sum_multi).  proj=1: the config-4 projection over
    (qty, price, disc, tax).  Returns (list of SUM columns, int64 counts or None)."""
    torch = _torch()
    if with_counts and counts is None:
        counts = torch.empty(n_groups, dtype=torch.int64, device=keys.device)
    dt, n, outs, cptr, optr, cnt = _multi_args(keys, cols, n_groups, proj, outs, counts if with_counts else None)
    st = _lib.repro_groupby_sum_multi(_dev(keys, "keys", torch.int32), cptr, len(cols), proj, n, n_groups, fold, dt,
                                      optr, cnt)
    _check(st, "repro_groupby_sum_multi")
    return outs, (counts if with_counts else None)


def groupby_sum_sparse(keys, vals, max_groups: int, fold: int = 3):
    """Reproducible GroupBy-SUM over arbitrary int64 or int32 keys
    (repro_groupby_sum_sparse / _i32).  Returns (distinct keys ascending as
    int64, their sums) as device tensors."""
    torch = _torch()
    dt = _dtype_code(vals)
    if keys.numel() != vals.numel():
        raise ValueError("keys and vals differ in length")
    ok = torch.empty(max_groups, dtype=torch.int64, device=vals.device)
    ov = torch.empty(max_groups, dtype=vals.dtype, device=vals.device)
    d = _i64()
    if keys.dtype == torch.int32:
        fn, name, kdt = _lib.repro_groupby_sum_sparse_i32, "repro_groupby_sum_sparse_i32", torch.int32
    else:
        fn, name, kdt = _lib.repro_groupby_sum_sparse, "repro_groupby_sum_sparse", torch.int64
    _check(fn(_dev(keys, "keys", kdt), _dev(vals, "vals"), keys.numel(), max_groups, fold, dt,
              _dev(ok, "out_keys", torch.int64), _dev(ov, "out_vals", vals.dtype), ctypes.byref(d)), name)
    return ok[: d.value], ov[: d.value]


def groupby_moments(keys, vals, n_groups: int, fold: int = 3):
    """Reproducible per-group SUM, AVG, sample VARIANCE, STDDEV and COUNT
    (repro_groupby_moments).  Returns a dict of device tensors."""
    torch = _torch()
    dt = _dtype_code(vals)
    if keys.numel() != vals.numel():
        raise ValueError("keys and vals differ in length")
    res = {k: torch.empty(n_groups, dtype=vals.dtype, device=vals.device) for k in ("sum", "avg", "var", "stddev")}
    res["count"] = torch.empty(n_groups, dtype=torch.int64, device=vals.device)
    _check(_lib.repro_groupby_moments(_dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel(), n_groups, fold,
                                      dt, *[_dev(res[k], k, vals.dtype) for k in ("sum", "avg", "var", "stddev")],
                                      _dev(res["count"], "count", torch.int64)), "repro_groupby_moments")
    return res


def sum(x, fold: int = 3, out=None):  # noqa: A001 -- the paper's operation name
    """Reproducible SUM of one array (repro_sum, blocking): a 1-element
    device tensor, the same bits as groupby_sum with every key 0."""
    torch = _torch()
    dt = _dtype_code(x)
    if out is None:
        out = torch.empty(1, dtype=x.dtype, device=x.device)
    _need(out, 1, "out")
    _check(_lib.repro_sum(_dev(x, "x"), x.numel(), fold, dt, _dev(out, "out", x.dtype)), "repro_sum")
    return out


def dot(x, y, fold: int = 3, out=None):
    """Reproducible dot product sum_i x_i (x) y_i (repro_dot, blocking)."""
    torch = _torch()
    dt = _dtype_code(x)
    if y.numel() != x.numel():
        raise ValueError("x and y differ in length")
    if out is None:
        out = torch.empty(1, dtype=x.dtype, device=x.device)
    _need(out, 1, "out")
    _check(_lib.repro_dot(_dev(x, "x"), _dev(y, "y", x.dtype), x.numel(), fold, dt, _dev(out, "out", x.dtype)),
           "repro_dot")
    return out


def dot_workspace_bytes(fold: int, dtype: int) -> int:
    return _lib.repro_dot_workspace_bytes(fold, dtype)


def dot_async(x, y, fold: int, out, workspace, status, stream=None):
    """Stream-ordered SUM (y None) or dot product (repro_dot_async)."""
    torch = _torch()
    dt = _dtype_code(x)
    if y is not None and y.numel() != x.numel():
        raise ValueError("x and y differ in length")
    _need(out, 1, "out")
    _need(status, 1, "status")
    wp, wb = _aligned_ptr(workspace)
    st = _lib.repro_dot_async(_dev(x, "x"), None if y is None else _dev(y, "y", x.dtype), x.numel(), fold, dt,
                              _dev(out, "out", x.dtype), wp, wb, _stream_ptr(stream),
                              _dev(status, "status", torch.int32))
    _check(st, "repro_dot_async")
    return out


def make_dot_workspace(fold: int, dtype: int, device="cuda"):
    torch = _torch()
    nbytes = dot_workspace_bytes(fold, dtype)
    if nbytes == 0:
        raise ReproError(EINVAL, "repro_dot_workspace_bytes")
    return torch.empty(nbytes + 256, dtype=torch.uint8, device=device)


def dot_table_views(workspace, fold: int, dtype: int):
    """(flags int32[1], kglob int32[1], slots int64[...]) views of the slot
    table inside a dot workspace (make_dot_workspace)."""
    torch = _torch()
    off, cnt = (_i64 * 3)(), (_i64 * 3)()
    _check(_lib.repro_dot_table(fold, dtype, off, cnt), "repro_dot_table")
    base = _aligned_ptr(workspace)[0] - workspace.data_ptr()
    return tuple(workspace[base + o: base + o + c * sz].view(dt)
                 for o, c, dt, sz in zip(off, cnt, (torch.int32, torch.int32, torch.int64), (4, 4, 8)))


def dot_deposit_async(x, y, fold: int, workspace, stream=None):
    dt = _dtype_code(x)
    if y is not None and y.numel() != x.numel():
        raise ValueError("x and y differ in length")
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_dot_deposit_async(_dev(x, "x"), None if y is None else _dev(y, "y", x.dtype), x.numel(),
                                        fold, dt, wp, wb, _stream_ptr(stream)), "repro_dot_deposit_async")


def dot_finish_async(fold: int, dtype: int, out, workspace, status, stream=None):
    torch = _torch()
    _need(out, 1, "out")
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_dot_finish_async(fold, dtype, _dev(out, "out"), wp, wb, _stream_ptr(stream),
                                       _dev(status, "status", torch.int32)), "repro_dot_finish_async")
    return out


def tune_get(fold: int, dtype: int) -> dict:
    """Path / depth settings (repro_tune_get): on-chip crossover (0 =
    capacity) and the widest one-pass partition id in bits."""
    a, b = _i32(), _i32()
    _check(_lib.repro_tune_get(fold, dtype, ctypes.byref(a), ctypes.byref(b)), "repro_tune_get")
    return {"onchip_max_groups": a.value, "onepass_bits": b.value}


def tune_set(fold: int, dtype: int, onchip_max_groups: int = 0, onepass_bits: int = 0):
    _check(_lib.repro_tune_set(fold, dtype, onchip_max_groups, onepass_bits), "repro_tune_set")


def autotune(n: int = 1 << 26, fold: int = 3, dtype: int = F64) -> dict:
    """Measure and set the crossovers on this GPU (repro_autotune)."""
    a, b = _i32(), _i32()
    _check(_lib.repro_autotune(n, fold, dtype, ctypes.byref(a), ctypes.byref(b)), "repro_autotune")
    return {"onchip_max_groups": a.value, "onepass_bits": b.value}


def multi_workspace_bytes(n: int, n_groups: int, ncols: int, proj: int, fold: int, dtype: int) -> int:
    return _lib.repro_groupby_multi_workspace_bytes(n, n_groups, ncols, proj, fold, dtype)


def make_multi_workspace(n, n_groups, ncols, proj, fold, dtype, device="cuda"):
    torch = _torch()
    nbytes = multi_workspace_bytes(n, n_groups, ncols, proj, fold, dtype)
    if nbytes == 0:
        raise ReproError(EINVAL, "repro_groupby_multi_workspace_bytes")
    return torch.empty(nbytes + 256, dtype=torch.uint8, device=device)


def groupby_sum_multi_async(keys, cols, n_groups: int, fold: int, proj: int, outs, counts, workspace, status,
                            stream=None):
    torch = _torch()
    dt, n, outs, cptr, optr, cnt = _multi_args(keys, cols, n_groups, proj, outs, counts)
    _need(status, 1, "status")
    wp, wb = _aligned_ptr(workspace)
    st = _lib.repro_groupby_sum_multi_async(_dev(keys, "keys", torch.int32), cptr, len(cols), proj, n, n_groups,
                                            fold, dt, optr, cnt, wp, wb, _stream_ptr(stream),
                                            _dev(status, "status", torch.int32))
    _check(st, "repro_groupby_sum_multi_async")
    return outs


def synth_generate(config: int, n: int, n_groups: int, r0: int = 0, seed: int | None = None, stream=None):
    """Seeded synthetic inputs of BASELINE config 0/1/2/4 generated on the
    device (same bits as synth.generate); returns (keys, [value columns])."""
    torch = _torch()
    from inputs.synth import SEED_BASE
    seed = SEED_BASE + config if seed is None else seed
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    cols = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4 if config == 4 else 1)]
    cptr = (_vp * len(cols))(*[_dev(c, "cols") for c in cols])
    _check(_lib.repro_synth_generate(config, seed, r0, n, n_groups, _dev(keys, "keys", torch.int32), cptr,
                                     _stream_ptr(stream)), "repro_synth_generate")
    return keys, cols


def multi_table_views(workspace, n: int, n_groups: int, ncols: int, proj: int, fold: int, dtype: int):
    """(flags int32[1], kglob int32[Gv], slots int64[...]) tensor views of the
    slot table inside a multi-column workspace (make_multi_workspace)."""
    torch = _torch()
    off = (_i64 * 3)()
    cnt = (_i64 * 3)()
    _check(_lib.repro_groupby_multi_table(n, n_groups, ncols, proj, fold, dtype, off, cnt), "repro_groupby_multi_table")
    base = _aligned_ptr(workspace)[0] - workspace.data_ptr()
    views = []
    for o, c, dt, sz in zip(off, cnt, (torch.int32, torch.int32, torch.int64), (4, 4, 8)):
        views.append(workspace[base + o: base + o + c * sz].view(dt))
    return tuple(views)


def groupby_multi_deposit_async(keys, cols, n_groups: int, fold: int, proj: int, workspace, stream=None):
    """Split form, step 1: deposit this rank's rows into the workspace's slot table."""
    torch = _torch()
    dt = _dtype_code(cols[0])
    cptr = (_vp * len(cols))(*[_dev(c, "cols") for c in cols])
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_groupby_multi_deposit_async(_dev(keys, "keys", torch.int32), cptr, len(cols), proj,
                                                  keys.numel(), n_groups, fold, dt, wp, wb, _stream_ptr(stream)),
           "repro_groupby_multi_deposit_async")


def groupby_multi_finish_async(n: int, n_groups: int, ncols: int, proj: int, fold: int, dtype: int, outs, counts,
                               workspace, status, stream=None):
    """Split form, step 3 (after the slot tables were all-reduced): read out."""
    torch = _torch()
    odt = torch.float64 if dtype == F64 else torch.float32
    optr = (_vp * len(outs))(*[_dev(o, "outs", odt) for o in outs])
    wp, wb = _aligned_ptr(workspace)
    _check(_lib.repro_groupby_multi_finish_async(n, n_groups, ncols, proj, fold, dtype, optr,
                                                 _dev(counts, "counts", torch.int64) if counts is not None else None,
                                                 wp, wb, _stream_ptr(stream), _dev(status, "status", torch.int32)),
           "repro_groupby_multi_finish_async")
    return outs


def baseline_atomic_sum(keys, vals, n_groups: int, variant: int = 0, accumulate_f64: bool = False, out=None,
                        stream=None):
    """Non-reproducible atomicAdd GroupBy on the same GPU (stream-ordered)."""
    torch = _torch()
    dt = _dtype_code(vals)
    odt = torch.float64 if (dt == F64 or accumulate_f64) else torch.float32
    if out is None:
        out = torch.empty(n_groups, dtype=odt, device=vals.device)
    _same_len(keys, vals)
    _need(out, n_groups, "out")
    st = _lib.repro_baseline_atomic_sum(_dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel(), n_groups,
                                        dt, variant, 1 if accumulate_f64 else 0, _dev(out, "out", odt),
                                        _stream_ptr(stream))
    _check(st, "repro_baseline_atomic_sum")
    return out


def measure_fp_add_rate(dtype: int, stream=None) -> float:
    """Measured correctly rounded adds per second of the value type's FP pipe
    on this GPU (the FP side of the roofline; repro_measure_fp_add_rate)."""
    r = ctypes.c_double(0.0)
    _check(_lib.repro_measure_fp_add_rate(dtype, ctypes.byref(r), _stream_ptr(stream)), "repro_measure_fp_add_rate")
    return r.value


def last_launch_count() -> int:
    return _lib.repro_last_launch_count()


def last_path() -> int:
    return _lib.repro_last_path()


def onchip_max_groups(fold: int, dtype: int) -> int:
    return _lib.repro_onchip_max_groups(fold, dtype)


def sweep_max_groups(fold: int, dtype: int) -> int:
    return _lib.repro_sweep_max_groups(fold, dtype)


def set_path_override(path: int):
    _lib.repro_set_path_override(path)


def set_kernel_variant(variant: int):
    """0 auto, 1 per-row atomics fed by the TMA ring, 2 k_table (register-fed
    counter table), 3 per-row atomics with register loads (bits never change)."""
    _lib.repro_set_kernel_variant(variant)


def set_route_mode(mode: int):
    """1: the routed one-pass kernel where the groups fit the SMs' tables
    (opt-in, measured slower); 0 (default): the two-pass sweep.  Bits never
    change."""
    _lib.repro_set_route_mode(mode)


def timing_enable(on: bool = True):
    """Bracket every kernel this thread enqueues with CUDA events (bench aid)."""
    _lib.repro_timing_enable(1 if on else 0)


def timing_collect() -> dict:
    """{kernel name: (launches, total device ms)} since the last collect."""
    names = (ctypes.c_char_p * 32)()
    counts = (_i32 * 32)()
    ms = (ctypes.c_double * 32)()
    k = _lib.repro_timing_collect(names, counts, ms, 32)
    return {names[i].decode(): (counts[i], ms[i]) for i in range(k)}


def release_cache():
    _lib.repro_release_cache()


class Accumulator:
    """n_groups device-resident repro<ScalarT, fold> states (repro_acc_*)."""

    def __init__(self, n_groups: int, fold: int = 3, dtype: int = F64):
        h = _vp()
        _check(_lib.repro_acc_create(ctypes.byref(h), n_groups, fold, dtype), "repro_acc_create")
        self._h = h
        self.n_groups, self.fold, self.dtype = n_groups, fold, dtype

    @property
    def _torch_dtype(self):
        torch = _torch()
        return torch.float64 if self.dtype == F64 else torch.float32

    def deposit(self, keys, vals):
        torch = _torch()
        if _dtype_code(vals) != self.dtype:
            raise TypeError("value dtype does not match the accumulator")
        _same_len(keys, vals)
        _check(_lib.repro_acc_deposit(self._h, _dev(keys, "keys", torch.int32), _dev(vals, "vals"), keys.numel()),
               "repro_acc_deposit")
        return self

    def merge(self, other: "Accumulator"):
        _check(_lib.repro_acc_merge(self._h, other._h), "repro_acc_merge")
        return self

    def finalize(self, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty(self.n_groups, dtype=self._torch_dtype, device="cuda")
        _need(out, self.n_groups, "out")
        _check(_lib.repro_acc_finalize(self._h, _dev(out, "out", self._torch_dtype)), "repro_acc_finalize")
        return out

    def export(self, state=None):
        torch = _torch()
        if state is None:
            state = torch.empty(self.n_groups * 2 * self.fold, dtype=self._torch_dtype, device="cuda")
        _need(state, self.n_groups * 2 * self.fold, "state")
        _check(_lib.repro_acc_export(self._h, _dev(state, "state", self._torch_dtype)), "repro_acc_export")
        return state

    def import_(self, state):
        _need(state, self.n_groups * 2 * self.fold, "state")
        _check(_lib.repro_acc_import(self._h, _dev(state, "state", self._torch_dtype)), "repro_acc_import")
        return self

    def reset(self):
        _check(_lib.repro_acc_reset(self._h), "repro_acc_reset")
        return self

    def top_levels(self, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty(self.n_groups, dtype=torch.int32, device="cuda")
        _need(out, self.n_groups, "k")
        _check(_lib.repro_acc_top_levels(self._h, _dev(out, "k", torch.int32)), "repro_acc_top_levels")
        return out

    def window_export(self, k_global, limbs=None):
        torch = _torch()
        if limbs is None:
            limbs = torch.empty(self.n_groups * self.fold * 2, dtype=torch.int64, device="cuda")
        _need(k_global, self.n_groups, "k_global")
        _need(limbs, self.n_groups * self.fold * 2, "limbs")
        _check(_lib.repro_acc_window_export(self._h, _dev(k_global, "k_global", torch.int32),
                                            _dev(limbs, "limbs", torch.int64)), "repro_acc_window_export")
        return limbs

    def window_import(self, k_global, limbs, g0: int = 0, count: int | None = None):
        torch = _torch()
        count = self.n_groups - g0 if count is None else count
        if g0 < 0 or count < 0 or g0 + count > self.n_groups:
            raise ValueError("group range outside the accumulator")
        _need(k_global, count, "k_global")
        _need(limbs, count * self.fold * 2, "limbs")
        _check(_lib.repro_acc_window_import_range(self._h, g0, count, _dev(k_global, "k_global", torch.int32),
                                                  _dev(limbs, "limbs", torch.int64)),
               "repro_acc_window_import_range")
        return self

    def close(self):
        if getattr(self, "_h", None):
            _lib.repro_acc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
