"""The device copy of the input generator (k_synth.cu) gives the same bits
as synth.py -- so oracle inputs generated on the host and bench inputs
generated on the device are the same rows."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import synth  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_09883_b200 as R
    return R


@pytest.mark.parametrize("config,G,r0", [(0, 16, 0), (1, 1024, 123456789), (2, 4096, 5), (4, 4, 1 << 29)])
def test_device_generator_matches_numpy(R, config, G, r0):
    n = 100003
    kd, cd = R.synth_generate(config, n, G, r0=r0)
    k, v = synth.generate(config, n=n, n_groups=G, r0=r0)
    assert np.array_equal(kd.cpu().numpy(), k)
    vs = v if config == 4 else (v,)
    for a, b in zip(cd, vs):
        assert a.cpu().numpy().tobytes() == np.ascontiguousarray(b).tobytes()
