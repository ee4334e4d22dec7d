"""Host-only checks of the f3 path / depth settings (repro_tune_get/set):
no GPU is needed, the calls only read and write the library's settings."""
import pytest

import paper_1802_09883_b200 as R


@pytest.fixture
def restore():
    saved = {(k, d): R.tune_get(k, d) for k in (1, 2, 3, 4) for d in (R.F32, R.F64)}
    yield
    for (k, d), v in saved.items():
        R.tune_set(k, d, v["onchip_max_groups"], v["onepass_bits"])


def test_defaults():
    assert R.tune_get(3, R.F64)["onepass_bits"] == 10
    assert R.tune_get(2, R.F32)["onepass_bits"] == 10


def test_round_trip(restore):
    R.tune_set(3, R.F64, 2048, 9)
    assert R.tune_get(3, R.F64) == {"onchip_max_groups": 2048, "onepass_bits": 9}
    assert R.tune_get(2, R.F64)["onchip_max_groups"] == 0  # per fold
    R.tune_set(3, R.F64, 0, 0)  # 0 bits leaves the depth unchanged
    assert R.tune_get(3, R.F64) == {"onchip_max_groups": 0, "onepass_bits": 9}


@pytest.mark.parametrize("args", [(0, R.F64, 0, 0), (5, R.F64, 0, 0), (3, 7, 0, 0), (3, R.F64, -1, 0),
                                  (3, R.F64, 0, 11), (3, R.F64, 0, -2)])
def test_invalid(restore, args):
    with pytest.raises(R.ReproError) as e:
        R.tune_set(*args)
    assert e.value.status == R.EINVAL


def test_autotune_rejects_bad_arguments_before_any_device_work():
    for args in ((1000, 3, R.F64), (1 << 20, 0, R.F64), (1 << 20, 3, 9)):
        with pytest.raises(R.ReproError) as e:
            R.autotune(*args)
        assert e.value.status == R.EINVAL
