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
    if cnt:
        acc.window_import(k[g0:g0 + cnt].contiguous(), mine[: cnt * width].contiguous(), g0=g0, count=cnt)
    local = torch.as_tensor(acc.finalize())
    part = torch.zeros(per, dtype=local.dtype, device=local.device)
    if cnt:
        part[:cnt] = local[g0:g0 + cnt]
    parts = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(parts, part, group=group)
    full = torch.cat(parts)[:G]
    out.copy_(full.to(out.device))
    return out


def allreduce_table(flags, kglob, slots, group=None):
    """Combine the per-rank absolute-level slot tables of the fused
    multi-column pass (repro_groupby_multi_table views): status bits OR-ed
    (NCCL has no bitwise reduction: one MAX over the four bits), window tops
    MAX, slot sums SUM -- integer operations, so every rank gets the same
    table whatever the reduction order."""
    bits = torch.stack([(flags[0] >> b) & 1 for b in range(4)]).to(torch.int32)
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    flags.copy_((bits * torch.tensor([1, 2, 4, 8], dtype=torch.int32, device=bits.device)).sum().reshape(1))
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
