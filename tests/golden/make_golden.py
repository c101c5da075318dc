"""Generate the golden fixtures from the UNCHANGED reference (build container only).

    python tests/golden/make_golden.py

For every case this runs a reference ``diffusekit.Session`` (numpy executor)
with a recorder attached (``tools/refcapture.py``) and writes, per case:

* the plan trace -- what the front end handed ``Session._execute`` -- and
* the final contents of every live store, as the reference computed them.

The GPU tests replay the traces through the B200 executor and compare against
these bytes; the CPU tests replay them through ``oracle/`` to pin the oracle.

``SPMV_CSR`` has no reference implementation.  The reference run
gets it as an injected builtin written here as plain Python loops (one float
accumulator per row, left to right), independent of ``oracle/``.
"""

from __future__ import annotations

import base64
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "tools"))
sys.path.insert(0, REPO)

from refcapture import import_reference, record_events  # noqa: E402

dk = import_reference()
sys.path.insert(0, "/root/reference/pkg/tests")
import stream_fuzz  # noqa: E402
from diffusekit.executor import default_builtins  # noqa: E402
from diffusekit.pipeline import Session, SessionConfig  # noqa: E402
from diffusekit.trace import gen_benchmark  # noqa: E402

from refcapture import attach_recorder  # noqa: E402
import workloads  # noqa: E402


def ref_spmv_csr(task, bufs):
    rowptr = bufs["a0"].reshape(-1)
    cols = bufs["a1"].reshape(-1)
    vals = bufs["a2"].reshape(-1)
    x = bufs["a3"].reshape(-1)
    y = bufs["a4"].reshape(-1)
    for i in range(rowptr.size - 1):
        acc = 0.0
        for j in range(int(rowptr[i]), int(rowptr[i + 1])):
            acc = acc + float(vals[j]) * float(x[int(cols[j])])
        y[i] = acc


def builtins():
    b = default_builtins()
    b["SPMV_CSR"] = ref_spmv_csr
    return b


def snapshot(session, ids):
    out = {}
    for s in ids:
        a = session.heap.get(s)
        out[str(s)] = {"shape": list(a.shape), "b64": base64.b64encode(a.tobytes()).decode()}
    return out


CONFIGS = {
    "fused": {},
    "unfused": {"fusion": False},
    "w2": {"window": 2},
    "notemp": {"temp_elim": False},
    "nomemo": {"memoize": False},
}


def case_from_events(name, events, cfg_name, init=None, dtypes=None):
    cfg = SessionConfig(**CONFIGS[cfg_name])
    session, report, trace = record_events(events, cfg, builtins=builtins(), init=init)
    trace.dtypes = dict(dtypes or {})
    trace.meta["name"] = f"{name}/{cfg_name}"
    return {"name": f"{name}/{cfg_name}", "trace": trace.to_json(), "final": snapshot(session, trace.live)}


def fuzz_case(seed, cfg_name):
    stream = stream_fuzz.generate_stream(seed)
    cfg = SessionConfig(**CONFIGS[cfg_name])
    session = Session(cfg, builtins=builtins())
    trace = attach_recorder(session)
    for sid in sorted(stream.stores):
        session.create_store(sid, stream.stores[sid])
    for i, t in enumerate(stream.tasks):
        session.submit(t)
        for sid in stream.drops.get(i, ()):
            session.drop_ref(sid)
    session.finish()
    trace.live = list(stream.live_ids)
    trace.meta["name"] = f"fuzz{seed}/{cfg_name}"
    return {"name": f"fuzz{seed}/{cfg_name}", "trace": trace.to_json(), "final": snapshot(session, trace.live)}


def write(path, cases):
    with gzip.open(path, "wt", compresslevel=9) as f:
        json.dump({"format": "dk-golden-1", "cases": cases}, f, separators=(",", ":"))
    print(f"wrote {path}: {len(cases)} cases")


def main():
    bench = []
    for name, kw in [
        ("stencil", dict(size=34, nodes=2, iters=3)),
        ("blackscholes_chain", dict(size=256, nodes=4, iters=5)),
        ("jacobi", dict(size=16, nodes=4, iters=3)),
        ("cg_like", dict(size=16, nodes=4, iters=3)),
    ]:
        for cfg in ("fused", "unfused", "w2", "notemp", "nomemo"):
            bench.append(case_from_events(name, gen_benchmark(name, **kw), cfg))
    for name, gen in [
        ("stencil_bands_n8_k2", lambda: workloads.stencil_bands(8, 2, 3)),
        ("stencil_bands_n6_k4", lambda: workloads.stencil_bands(6, 4, 2)),
        ("cg_csr_8x8_k2", lambda: workloads.cg_csr(8, 8, 2, 6)),
        ("cg_csr_6x12_k4", lambda: workloads.cg_csr(6, 12, 4, 4)),
        ("pcg_csr_8x8_k2", lambda: workloads.pcg_csr(8, 8, 2, 6)),
    ]:
        for cfg in ("fused", "unfused"):
            ev, init, dt = gen()
            bench.append(case_from_events(name, ev, cfg, init, dt))
    write(os.path.join(HERE, "bench_small.json.gz"), bench)

    fuzz = []
    for seed in range(250):
        for cfg in ("fused", "unfused", "w2"):
            fuzz.append(fuzz_case(seed, cfg))
    write(os.path.join(HERE, "fuzz250.json.gz"), fuzz)


if __name__ == "__main__":
    main()
