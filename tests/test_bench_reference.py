"""The bench contract's reference arm runs on the host (the CPU oracle): the
JSON line it prints carries the contract's keys.  Config 0 (2^16 rows) and
the f4 SUM workload, one step each -- seconds on CPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", [0, 5])
def test_reference_arm_prints_the_contract_line(config):
    extra = ["--rows", str(1 << 16)] if config == 5 else []
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          str(config), "--steps", "1", "--warmup", "1", *extra],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "rows/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    # the oracle arm never maps the product library
    assert d["repo_libs_mapped"] is not None
    assert not any("librepro_b200" in p for p in d["repo_libs_mapped"]), d["repo_libs_mapped"]
    assert any("liboracle" in p for p in d["repo_libs_mapped"]), d["repo_libs_mapped"]


def test_roofline_traffic_lookup_matches_workload_launch_and_kernel():
    """roofline.traffic comes from a committed ncu --set full capture only when config, group count, launch size and
    kernel all match; every source it names is a tracked profile holding the dram__bytes metrics."""
    sys.path.insert(0, ROOT)
    import bench
    t, src = bench.ncu_traffic(1, 1024, 1 << 27, "table_accumulate")
    assert t and 1.0 <= t / ((1 << 27) * 12) < 1.05 and os.path.exists(os.path.join(ROOT, src))
    assert bench.ncu_traffic(1, 1024, 1 << 26, "table_accumulate") == (None, None)
    assert bench.ncu_traffic(1, 1024, 1 << 27, "fold") == (None, None)
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
        for key, e in json.load(fh)["r2"].items():
            with open(os.path.join(ROOT, e["source"])) as ph:
                text = ph.read()
            assert "dram__bytes_read.sum" in text and "dram__bytes_write.sum" in text, key
