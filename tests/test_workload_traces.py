"""f4: the harness workloads as JSON-lines traces in the reference's own format (trace.py:73-192).

Each new stream (row-band stencil with residual, CSR CG, Jacobi-PCG) is written
with the reference's printer plus ``init`` / ``dtype`` annotations on its
``create_store`` lines and read back with the reference's parser: identical
events, identical annotations, the reference CLI (``diffusekit analyze`` /
``canon``) accepts the file and reports the same fusion plan, and a reference
Session run from the parsed file ends with the same heap as one from the
generator.
"""

import io
import os
import sys
from contextlib import redirect_stdout

import numpy as np
import pytest

from conftest import REPO, reference_available

pytestmark = pytest.mark.skipif(reference_available() is None, reason="reference not importable")

CASES = [("stencil", (8, 2, 3)), ("cg", (8, 8, 2, 4)), ("pcg", (8, 8, 2, 4)), ("cg", (6, 12, 4, 3))]


@pytest.fixture(scope="module")
def W():
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import workloads

    return workloads


def _gen(W, kind, args):
    return {"stencil": W.stencil_bands, "cg": W.cg_csr, "pcg": W.pcg_csr}[kind](*args)


def _run(events, init, cfg=None):
    from diffusekit.pipeline import SessionConfig

    from refcapture import record_events
    sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
    from make_golden import builtins

    session, report, trace = record_events(events, cfg or SessionConfig(), builtins=builtins(), init=init)
    return session, report


@pytest.mark.parametrize("kind,args", CASES)
def test_jsonl_round_trip(W, kind, args, tmp_path):
    events, init, dtypes = _gen(W, kind, args)
    text = W.write_jsonl(events, init, dtypes)
    ev2, init2, dt2 = W.read_jsonl(text)
    assert ev2 == list(events)
    assert init2 == init and dt2 == dtypes
    assert W.write_jsonl(ev2, init2, dt2) == text
    # the reference CLI reads the file and reports the same fusion plan as a direct run
    path = tmp_path / f"{kind}.jsonl"
    path.write_text(text)
    from diffusekit import cli
    from diffusekit.pipeline import Session, SessionConfig, run_events

    buf = io.StringIO()
    with redirect_stdout(buf):
        assert cli.main(["analyze", str(path), "--json-report", str(tmp_path / "r.json")]) == 0
        assert cli.main(["canon", str(path)]) == 0
    import json

    rep = json.loads((tmp_path / "r.json").read_text())
    direct = run_events(Session(SessionConfig(execute=False)), list(events))
    assert rep["fused_prefixes"] == list(direct.fused_prefixes)
    # executing the parsed file gives the generator's heap
    s1, r1 = _run(list(events), init)
    s2, r2 = _run(ev2, init2)
    assert list(r1.fused_prefixes) == list(r2.fused_prefixes)
    for sid in s1.live_store_ids():
        assert np.array_equal(s1.heap.get(sid), s2.heap.get(sid), equal_nan=True)
