import base64
import gzip
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as f:
        return json.load(f)["cases"]


def golden_arrays(case):
    out = {}
    for s, v in case["final"].items():
        out[int(s)] = np.frombuffer(base64.b64decode(v["b64"]), dtype=np.float64).reshape(v["shape"])
    return out


def same_bits(a, b):
    """Byte equality with every NaN treated as equal (payloads differ across ISAs)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not (na == nb).all():
        return False
    return a[~na].tobytes() == b[~nb].tobytes()


@pytest.fixture(scope="session")
def bench_cases():
    return load_golden("bench_small.json.gz")


@pytest.fixture(scope="session")
def fuzz_cases():
    return load_golden("fuzz250.json.gz")


def reference_available():
    for cand in ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "diffusekit")):
            return cand
    return None
