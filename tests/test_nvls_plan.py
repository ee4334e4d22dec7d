"""Plan and layout of the in-switch (NVLS) slot-table all-reduce (SURVEY.md
8(f) f4), checked on CPU: the per-rank slices cover every word exactly once,
the table regions meet multimem's natural alignment, and without multicast
support the exchange falls back to NCCL / gloo collectives (NvlsWorkspace
is None)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_1802_09883_b200 import dist as rdist


@pytest.mark.parametrize("n", [0, 1, 7, 1000, (1 << 20) + 3])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_slices_cover_every_word_once(n, world):
    hit = np.zeros(n, np.int32)
    for lo, hi in rdist.nvls_slices(n, world):
        assert 0 <= lo <= hi <= n
        hit[lo:hi] += 1
    assert (hit == 1).all()


@pytest.mark.parametrize("G,K,dt", [(1, 1, 1), (1024, 3, 1), (5000, 3, 1), (1 << 20, 2, 0), (33, 4, 0)])
def test_table_regions_are_naturally_aligned(G, K, dt):
    import paper_1802_09883_b200 as R
    off, cnt = R.table_layout(1 << 20, G, K, dt)
    assert off[0] % 4 == 0 and off[1] % 4 == 0 and off[2] % 8 == 0  # b32 status, s32 tops, u64 slots
    assert cnt[0] == 1 and cnt[1] == G and cnt[2] == G * ((25 if dt == 1 else 7) + K) * 2
    assert off[0] + 4 <= off[1] and off[1] + 4 * G <= off[2]
    assert off[2] + 8 * cnt[2] <= R.workspace_bytes(1 << 20, G, K, dt)


def test_no_multicast_means_collective_fallback():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29731"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        assert rdist.NvlsWorkspace.create(1 << 20) is None
    finally:
        dist.destroy_process_group()
