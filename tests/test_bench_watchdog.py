"""bench.ExtrasWatchdog: a hang after the headline measurement still yields exactly one JSON line."""

import json
import os
import subprocess
import sys

from conftest import REPO

_SCRIPT = r"""
import sys, time
sys.path.insert(0, {repo!r})
import bench
out = {{"metric": "m", "value": 1.5, "unit": "iter/s", "workloads": {{}}}}
w = bench.ExtrasWatchdog(0, out, {budget})
out["workloads"]["stencil"] = {{"fused_iter_s": 2.0}}
time.sleep({sleep})      # a hung extra
w.finish()
w.finish()               # printed once
"""


def _run(budget, sleep):
    r = subprocess.run([sys.executable, "-c", _SCRIPT.format(repo=REPO, budget=budget, sleep=sleep)],
                       capture_output=True, text=True, timeout=120, env=dict(os.environ))
    return r.returncode, [json.loads(x) for x in r.stdout.strip().splitlines() if x.strip()]


def test_watchdog_prints_once_when_extras_hang():
    rc, lines = _run(budget=1.0, sleep=30)
    assert rc == 0 and len(lines) == 1
    assert lines[0]["value"] == 1.5 and lines[0]["extras_timeout_s"] == 1.0
    assert lines[0]["workloads"]["stencil"]["fused_iter_s"] == 2.0


def test_watchdog_normal_path_prints_once():
    rc, lines = _run(budget=60.0, sleep=0)
    assert rc == 0 and len(lines) == 1 and "extras_timeout_s" not in lines[0]
