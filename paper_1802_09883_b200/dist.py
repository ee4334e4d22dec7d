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


def shard_rows(n: int, world: int, rank: int):
    """Contiguous row range [r0, r1) of `rank` (rows are independent units)."""
    r0 = n * rank // world
    r1 = n * (rank + 1) // world
    return r0, r1
