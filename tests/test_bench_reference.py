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
