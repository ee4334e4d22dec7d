"""Multi-GPU combination of per-rank accumulator tables.

One process per GPU; rows shard across ranks (each rank deposits its own
rows).  The exchange is integer-only, so the result is bit-identical for any
rank count and any NCCL algorithm (ring / tree / NVLS):

  1. k   = top lattice index of every group (repro_acc_top_levels)
  2. all-reduce MAX on k                      -> global window tops
  3. limbs = level sums realigned to the global tops (the paper's level
     demotion), carry-split into [0, 2^32) / high parts
     (repro_acc_window_export)
  4. all-reduce SUM on limbs (exact integer addition)
  5. canonicalise into every rank's handle (repro_acc_window_import,
     Alg. 1 lines 17-21)

`acc` is any object with top_levels() / window_export(k) / window_import(k,
limbs) -- the CUDA Accumulator in production; the CPU gloo tests pass a
test double so this host logic is exercised without a GPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def allreduce_state(acc, group=None):
    """Combine every rank's accumulator into the global state (in place)."""
    k = acc.top_levels()
    dist.all_reduce(k, op=dist.ReduceOp.MAX, group=group)
    limbs = acc.window_export(k)
    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)
    acc.window_import(k, limbs)
    return acc


def reduce_scatter_finalize(acc, out, group=None):
    """SURVEY.md 8(e) with a reduce-scatter by contiguous group range (less
    traffic than allreduce_state at high group counts):

      1. all-reduce MAX on the window tops;
      2. realign to the global tops (window_export);
      3. reduce-scatter SUM of the limbs: rank r receives groups
         [r * P, (r + 1) * P), P = ceil(G / world);
      4. canonicalise and finalise the owned range (window_import range form);
      5. all-gather the finalised values into `out` (every rank, all groups).

    Integer SUM / MAX only, so `out` is bit-identical for any rank count.
    Afterwards each rank's handle holds the combined state of ITS range only.
    Backends without reduce-scatter (gloo) take the all-reduce + slice form of
    step 3 (same integers)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    G, K = acc.n_groups, acc.fold
    k = acc.top_levels()
    dist.all_reduce(k, op=dist.ReduceOp.MAX, group=group)
    limbs = acc.window_export(k)
    per = -(-G // world)
    width = 2 * K
    padded = torch.zeros(per * world * width, dtype=torch.int64, device=limbs.device)
    padded[: G * width].copy_(limbs)
    if dist.get_backend(group) == "nccl":
        mine = torch.empty(per * width, dtype=torch.int64, device=limbs.device)
        dist.reduce_scatter_tensor(mine, padded, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(padded, op=dist.ReduceOp.SUM, group=group)
        mine = padded[rank * per * width:(rank + 1) * per * width].clone()
    g0 = rank * per
    cnt = max(0, min(per, G - g0))
    # every group outside this rank's range is set to the zero state, so the
    # read-out below can only fail (ERANGE) on the combined groups this rank
    # owns; the failure is shared through an all-reduce before anyone raises
    # (every rank reaches every collective)
    zk = torch.zeros(G, dtype=torch.int32, device=limbs.device)
    zl = torch.zeros(G * width, dtype=torch.int64, device=limbs.device)
    acc.window_import(zk, zl)
    if cnt:
        acc.window_import(k[g0:g0 + cnt].contiguous(), mine[: cnt * width].contiguous(), g0=g0, count=cnt)
    err = 0
    try:
        local = torch.as_tensor(acc.finalize())
    except Exception as e:  # noqa: BLE001 -- the status is shared, then re-raised on every rank
        err, local, exc = 1, torch.zeros(G, dtype=out.dtype, device=limbs.device), e
    flag = torch.tensor([err], dtype=torch.int32, device=limbs.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    part = torch.zeros(per, dtype=local.dtype, device=local.device)
    if cnt:
        part[:cnt] = local[g0:g0 + cnt]
    parts = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(parts, part, group=group)
    if int(flag.item()):
        if err:
            raise exc
        raise RuntimeError("reduce_scatter_finalize: the read-out failed on another rank")
    full = torch.cat(parts)[:G]
    out.copy_(full.to(out.device))
    return out


def _flag_bits_max(flags, group=None):
    """Bitwise OR of the 4 status bits over the ranks (NCCL has no bitwise
    reduction: MAX per bit)."""
    bits = torch.stack([(flags[0] >> b) & 1 for b in range(4)]).to(torch.int32)
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    flags.copy_((bits * torch.tensor([1, 2, 4, 8], dtype=torch.int32, device=bits.device)).sum().reshape(1))


def nvls_slices(n: int, world: int):
    """The words of an n-word region each rank reduces through the switch
    (k_nvls.cu slice): contiguous, disjoint, covering [0, n)."""
    per = -(-n // world) if world else 0
    return [(min(n, r * per), min(n, min(n, r * per) + per)) for r in range(world)]


class NvlsWorkspace:
    """A workspace in symmetric memory that every rank also maps at one
    multicast address (NVSwitch NVLS), for repro_nvls_table_allreduce_async.
    create() returns None where multicast is unavailable (CPU, gloo, PCIe
    GPUs, no NVSwitch): the callers then exchange with NCCL collectives."""

    def __init__(self, buf, handle):
        self.buf, self.handle = buf, handle
        aligned = (buf.data_ptr() + 255) // 256 * 256
        self.mc = handle.multicast_ptr + (aligned - buf.data_ptr())

    @staticmethod
    def create(nbytes: int, group=None):
        try:
            if not torch.cuda.is_available() or dist.get_backend(group) != "nccl":
                return None
            import torch.distributed._symmetric_memory as symm
            dev = torch.cuda.current_device()
            if not torch._C._distributed_c10d._SymmetricMemory.has_multicast_support(
                    torch._C._autograd.DeviceType.CUDA, dev):
                return None
            buf = symm.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{dev}")
            handle = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
            if not handle.multicast_ptr:
                return None
            return NvlsWorkspace(buf, handle)
        except Exception:  # noqa: BLE001 -- any failure means "no NVLS here"
            return None

    def allreduce_table(self, R, offsets, counts, group=None, stream=None):
        """Barrier (every rank's deposit done), in-switch OR / MAX / ADD of the
        table, barrier (every rank's multicast stores visible)."""
        self.handle.barrier(channel=0)
        R.nvls_table_allreduce_async(self.mc, offsets, counts, dist.get_rank(group), dist.get_world_size(group),
                                     stream)
        self.handle.barrier(channel=0)


def groupby_sum_dist(R, keys, vals, n_groups, fold, out, workspace, status, group=None, stream=None,
                     reduce_scatter=None, nvls=None):
    """Single-column GroupBy over the rows of all ranks, stream-ordered end to
    end: deposit the local rows into the workspace's
    absolute-level slot table, combine the status bits (OR) and window tops
    (MAX), then either

      * all-reduce the slot table (SUM) and read every group out on every rank
        (small group counts), or
      * take the K slot words under the global tops (the realignment), reduce-
        scatter them by contiguous group range (SUM), read out the owned range
        and all-gather the outputs (large group counts: 2K int64 per group
        reduced instead of the whole table).

    Integer SUM / MAX only: the bits equal the one-GPU result for any rank
    count and any reduction order.  No host synchronisation: the collectives
    are ordered on the current stream.  Every rank ends with the same status
    word (the deposit bits are combined first; a read-out ERANGE is shared by a
    MIN over the codes, whose precedence EKEY > EDOM > ERANGE is -2 > -3 > -4)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    G, K = n_groups, fold
    dt = R.F64 if vals.dtype == torch.float64 else R.F32
    n = keys.numel()
    if nvls is not None:  # exchange A through the switch; `workspace` must be nvls.buf
        R.groupby_deposit_async(keys, vals, G, K, nvls.buf, stream)
        off, cnt = R.table_layout(n, G, K, dt)
        nvls.allreduce_table(R, off, cnt, group, stream)
        R.groupby_finish_async(n, G, K, dt, out, nvls.buf, status, stream)
        return out
    R.groupby_deposit_async(keys, vals, G, K, workspace, stream)
    flags, kglob, slots = R.groupby_table_views(workspace, n, G, K, dt)
    _flag_bits_max(flags, group)
    dist.all_reduce(kglob, op=dist.ReduceOp.MAX, group=group)
    if reduce_scatter is None:
        reduce_scatter = G >= 4096 and world > 1
    if not reduce_scatter:
        dist.all_reduce(slots, op=dist.ReduceOp.SUM, group=group)
        R.groupby_finish_async(n, G, K, dt, out, workspace, status, stream)
    else:
        per = -(-G // world)
        width = 2 * K
        limbs = torch.zeros(per * world * width, dtype=torch.int64, device=slots.device)
        R.groupby_window_limbs_async(n, G, K, dt, kglob, limbs, workspace, stream)
        if dist.get_backend(group) == "nccl":
            mine = torch.empty(per * width, dtype=torch.int64, device=limbs.device)
            dist.reduce_scatter_tensor(mine, limbs, op=dist.ReduceOp.SUM, group=group)
        else:  # gloo has no reduce-scatter: all-reduce + slice (same integers)
            dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)
            mine = limbs[rank * per * width:(rank + 1) * per * width].contiguous()
        g0 = rank * per
        cnt = max(0, min(per, G - g0))
        part = torch.zeros(per, dtype=out.dtype, device=out.device)
        R.groupby_finish_limbs_async(n, G, K, dt, g0, cnt, kglob[g0:g0 + cnt], mine[: cnt * width], part[:cnt],
                                     workspace, status, stream)
        parts = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(parts, part, group=group)
        out.copy_(torch.cat(parts)[:G])
    dist.all_reduce(status, op=dist.ReduceOp.MIN, group=group)
    return out


def allreduce_table(flags, kglob, slots, group=None):
    """Combine the per-rank absolute-level slot tables of the fused
    multi-column pass (repro_groupby_multi_table views): status bits OR-ed
    (NCCL has no bitwise reduction: one MAX over the four bits), window tops
    MAX, slot sums SUM -- integer operations, so every rank gets the same
    table whatever the reduction order."""
    _flag_bits_max(flags, group)
    dist.all_reduce(kglob, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(slots, op=dist.ReduceOp.SUM, group=group)


def groupby_sum_multi_dist(R, keys, cols, n_groups, fold, proj, outs, counts, workspace, status, group=None,
                           stream=None):
    """Multi-column GroupBy over the rows of all ranks: deposit locally,
    all-reduce the slot tables, read out on every rank."""
    dt = R.F64 if cols[0].dtype == torch.float64 else R.F32
    n = keys.numel()
    R.groupby_multi_deposit_async(keys, cols, n_groups, fold, proj, workspace, stream)
    flags, kglob, slots = R.multi_table_views(workspace, n, n_groups, len(cols), proj, fold, dt)
    allreduce_table(flags, kglob, slots, group)
    R.groupby_multi_finish_async(n, n_groups, len(cols), proj, fold, dt, outs, counts, workspace, status, stream)
    return outs


def dot_dist(R, x, y, fold, out, workspace, status, group=None, stream=None):
    """Single-array SUM (y None) or dot product over the elements of all
    ranks: deposit the local shard, all-reduce the slot table, read out on
    every rank (same bits as one GPU over the concatenated arrays)."""
    dt = R.F64 if x.dtype == torch.float64 else R.F32
    R.dot_deposit_async(x, y, fold, workspace, stream)
    flags, kglob, slots = R.dot_table_views(workspace, fold, dt)
    allreduce_table(flags, kglob, slots, group)
    R.dot_finish_async(fold, dt, out, workspace, status, stream)
    return out


def shard_rows(n: int, world: int, rank: int):
    """Contiguous row range [r0, r1) of `rank` (rows are independent units)."""
    r0 = n * rank // world
    r1 = n * (rank + 1) // world
    return r0, r1
