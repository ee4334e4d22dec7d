"""The in-switch (NVLS) slot-table exchange on the GPU: a one-rank NCCL group
over symmetric memory with a multicast mapping (when the box offers it; the
test is skipped otherwise).  multimem.ld_reduce over one rank is the
identity, so the result must equal the one-GPU GroupBy and the oracle bit for
bit; the LDGMC / STGMC instructions run on the hardware."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402  (test infrastructure)


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


def test_nvls_exchange_one_rank(R):
    import torch.distributed as dist
    from paper_1802_09883_b200 import dist as rdist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29733")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        G, K, n = 1024, 3, 1 << 20
        nv = rdist.NvlsWorkspace.create(R.workspace_bytes(n, G, K, R.F64))
        if nv is None:
            pytest.skip("no multicast (NVLS) support on this GPU / driver")
        rng = np.random.default_rng(5)
        keys = rng.integers(0, G, n, dtype=np.int32)
        vals = rng.standard_normal(n) * np.exp2(rng.integers(-30, 31, n))
        out = torch.empty(G, dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        rdist.groupby_sum_dist(R, torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, K, out, None, st,
                               nvls=nv)
        torch.cuda.synchronize()
        rc, ref = O.groupby_sum(keys, vals, G, K)
        assert rc == 0 and st.item() == 0
        assert out.cpu().numpy().tobytes() == ref.tobytes()
    finally:
        dist.destroy_process_group()
