"""GPU checks of the f3 runtime path / depth selection (repro_autotune,
repro_tune_set): the autotuner runs and sets sane crossovers, and the result
bits do not depend on the path or depth chosen -- every setting is compared
with the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from inputs import synth  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


@pytest.fixture
def restore(R):
    saved = {(k, d): R.tune_get(k, d) for k in (1, 2, 3, 4) for d in (R.F32, R.F64)}
    yield
    for (k, d), v in saved.items():
        R.tune_set(k, d, v["onchip_max_groups"], v["onepass_bits"])


def rows(n, G, dtype, seed):
    keys, vals = synth.generate(2, n=n, n_groups=G, seed=seed)
    return keys, vals.astype(dtype)


def run(R, keys, vals, G, K):
    out = R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, K)
    torch.cuda.synchronize()
    return out.cpu().numpy(), R.last_path()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_autotune_sets_sane_crossovers(R, restore, dtype):
    dt = R.F64 if dtype == np.float64 else R.F32
    K = 3 if dtype == np.float64 else 2
    res = R.autotune(1 << 22, K, dt)
    cap = R.onchip_max_groups(K, dt)
    assert 1024 <= res["onchip_max_groups"] <= cap
    assert 1 <= res["onepass_bits"] <= 10
    assert R.tune_get(K, dt) == res
    # the tuned settings still give the oracle's bits on both sides of the crossover
    for G in (1024, 2048, 4096, 1 << 18):
        keys, vals = rows(300007, G, dtype, 40 + G % 7)
        got, _ = run(R, keys, vals, G, K)
        rc, ref = O.groupby_sum(keys, vals, G, K)
        assert rc == O.OK and got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("G", [2048, 4096])
def test_onchip_crossover_setting_changes_path_not_bits(R, restore, G):
    keys, vals = rows(500009, G, np.float64, 3)
    R.tune_set(3, R.F64, 1024, 0)
    part, p1 = run(R, keys, vals, G, 3)
    R.tune_set(3, R.F64, 0, 0)
    onchip, p0 = run(R, keys, vals, G, 3)
    assert (p1, p0) == (1, 0)
    rc, ref = O.groupby_sum(keys, vals, G, 3)
    assert rc == O.OK and part.tobytes() == onchip.tobytes() == ref.tobytes()


@pytest.mark.parametrize("dtype,K,G", [(np.float64, 3, 1 << 19), (np.float64, 3, 1 << 20),
                                       (np.float32, 2, 1 << 19), (np.float64, 2, 1 << 13)])
def test_depth_setting_changes_passes_not_bits(R, restore, dtype, K, G):
    """Partition ids of log2(G / 1024) bits: one pass (multisplit or wide
    scatter) vs two passes give the same bits."""
    dt = R.F64 if dtype == np.float64 else R.F32
    keys, vals = rows(1 << 21, G, dtype, 5)
    pbits = (G // 1024 - 1).bit_length()
    outs = []
    for bits in (10, max(1, pbits - 1)):
        R.tune_set(K, dt, 1024, bits)
        got, path = run(R, keys, vals, G, K)
        assert path == 1
        outs.append(got)
    assert outs[0].tobytes() == outs[1].tobytes()
    sel = np.unique(np.concatenate([[0, G - 1], np.random.default_rng(1).integers(0, G, 200)])).astype(np.int32)
    rc, ref = O.groupby_sum_select(keys, vals, G, K, sel)
    assert rc == O.OK and outs[0][sel].tobytes() == ref.tobytes()


def test_workspace_follows_the_path(R, restore):
    """A workspace sized before a crossover change is too small for the
    partitioned path: loud ENOMEM, never a wrong result."""
    G, K, n = 4096, 3, 100000
    keys, vals = rows(n, G, np.float64, 9)
    ws_on = R.make_workspace(n, G, K, R.F64)
    R.tune_set(K, R.F64, 1024, 0)
    ws_part = R.make_workspace(n, G, K, R.F64)
    assert ws_part.numel() > ws_on.numel()
    out = torch.empty(G, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    dk, dv = torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda()
    with pytest.raises(R.ReproError) as e:
        R.groupby_sum_async(dk, dv, G, K, out, ws_on, status)
    assert e.value.status == R.ENOMEM
    R.groupby_sum_async(dk, dv, G, K, out, ws_part, status)
    torch.cuda.synchronize()
    rc, ref = O.groupby_sum(keys, vals, G, K)
    assert status.item() == 0 and out.cpu().numpy().tobytes() == ref.tobytes()
