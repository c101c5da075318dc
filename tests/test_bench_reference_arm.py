"""The reference arm of bench.py on CPU: `--impl reference` runs the unmodified reference Session on a
bounded sample and prints the contract's JSON line (impl, metric/unit of our arm, cpu_baseline, e2e)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO


@pytest.mark.skipif(not os.path.isdir(os.path.join(REPO, "baseline", "_ref", "diffusekit")),
                    reason="reference not installed under baseline/_ref")
def test_reference_arm_prints_contract_line():
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "iter/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["n_gpus"] == 1 and line["steps"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == line["value"] and cb["cores"] >= 1 and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "iter/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["metric"].startswith("fused iters/sec")
