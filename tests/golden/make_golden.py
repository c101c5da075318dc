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


def edge_streams():
    """Hand-written streams for the binding edge cases the benchmarks do not reach.

    Each returns the reference's own trace events: clamped (ragged) tiles,
    empty sub-stores (ir.py:264-267), rank-0 nests, whole-store writes by
    several points, 2-D ragged tiles, scalar-valued reductions (kernels.py:765).
    """
    from diffusekit.trace import CreatePartition, CreateStore, DropRef, Flush, TaskEvent

    def ident(r):
        return (tuple(tuple(1 if i == j else 0 for j in range(r)) for i in range(r)), (0,) * r)

    out = {}
    # 1-D ragged: store 10, tile 4, launch 3 -> last tile [8, 10)
    ev = [CreateStore(0, (10,)), CreateStore(1, (10,)), CreateStore(2, (10,)), CreateStore(3, ()), CreateStore(4, (10,))]
    ev += [CreatePartition(i, i, "tiling", (4,), (0,), ident(1)) for i in (0, 1, 2, 4)]
    ev += [CreatePartition(3, 3, "none")]
    for _ in range(2):
        ev += [TaskEvent("ADD", (3,), ((0, 0, "R"), (1, 1, "R"), (4, 4, "W"))),
               TaskEvent("MULT", (3,), ((4, 4, "R"), (2, 2, "W")), (("s", 0.5),)),
               TaskEvent("DOT", (3,), ((2, 2, "R"), (0, 0, "R"), (3, 3, "Rd"))),
               TaskEvent("MAX", (3,), ((2, 2, "R"), (1, 1, "R"), (0, 0, "W"))),
               Flush()]
    out["edge_ragged_1d"] = ev
    # empty sub-stores: store 6, tile 4, launch 3 -> point 2 is [6, 6)
    ev = [CreateStore(0, (6,)), CreateStore(1, (6,)), CreateStore(2, ())]
    ev += [CreatePartition(0, 0, "tiling", (4,), (0,), ident(1)), CreatePartition(1, 1, "tiling", (4,), (0,), ident(1)),
           CreatePartition(2, 2, "none")]
    for _ in range(2):
        ev += [TaskEvent("NEG", (3,), ((0, 0, "R"), (1, 1, "W"))),
               TaskEvent("DOT", (3,), ((1, 1, "R"), (1, 1, "R"), (2, 2, "Rd"))),
               TaskEvent("AXPY_RATIO", (3,), ((1, 1, "R"), (0, 0, "RW"), (2, 2, "R"), (2, 2, "R"))),
               Flush()]
    out["edge_empty_tiles"] = ev
    # 2-D ragged: store (5, 7), tile (2, 3), launch (3, 3)
    ev = [CreateStore(0, (5, 7)), CreateStore(1, (5, 7)), CreateStore(2, (5, 7)), CreateStore(3, ())]
    ev += [CreatePartition(i, i, "tiling", (2, 3), (0, 0), ident(2)) for i in range(3)]
    ev += [CreatePartition(3, 3, "none")]
    for _ in range(2):
        ev += [TaskEvent("SUB", (3, 3), ((0, 0, "R"), (1, 1, "R"), (2, 2, "W"))),
               TaskEvent("MIN", (3, 3), ((2, 2, "R"), (0, 0, "R"), (1, 1, "W"))),
               TaskEvent("SUM", (3, 3), ((1, 1, "R"), (3, 3, "Rd"))),
               TaskEvent("AXPY", (3, 3), ((1, 1, "R"), (0, 0, "RW")), (("w", -1.0),)),
               Flush()]
    out["edge_ragged_2d"] = ev
    # rank-0 stores: FILL by every point, scalar-valued DOT/SUM (rank-0 nests), ratio reads
    ev = [CreateStore(0, ()), CreateStore(1, ()), CreateStore(2, ()), CreateStore(3, (8,)), CreateStore(4, (8,))]
    ev += [CreatePartition(i, i, "none") for i in range(3)]
    ev += [CreatePartition(3, 3, "tiling", (4,), (0,), ident(1)), CreatePartition(4, 4, "tiling", (4,), (0,), ident(1))]
    for _ in range(2):
        ev += [TaskEvent("FILL", (2,), ((0, 0, "W"),), (("s", 3.0),)),
               TaskEvent("DOT", (2,), ((0, 0, "R"), (0, 0, "R"), (1, 1, "Rd"))),
               TaskEvent("SUM", (2,), ((0, 0, "R"), (2, 2, "Rd"))),
               TaskEvent("XPBY_RATIO", (2,), ((3, 3, "R"), (4, 4, "RW"), (1, 1, "R"), (2, 2, "R"))),
               Flush()]
    out["edge_rank0"] = ev
    # divisions by zero and NaN / inf propagation through min/max/neg
    ev = [CreateStore(0, (6,)), CreateStore(1, (6,)), CreateStore(2, (6,)), CreateStore(3, (6,))]
    ev += [CreatePartition(i, i, "tiling", (3,), (0,), ident(1)) for i in range(4)]
    ev += [TaskEvent("FILL", (2,), ((3, 3, "W"),), (("s", 0.0),)),
           TaskEvent("DIV", (2,), ((0, 0, "R"), (3, 3, "R"), (1, 1, "W"))),
           TaskEvent("SUB", (2,), ((1, 1, "R"), (1, 1, "R"), (2, 2, "W"))),
           TaskEvent("MIN", (2,), ((2, 2, "R"), (0, 0, "R"), (3, 3, "W"))),
           TaskEvent("MAX", (2,), ((1, 1, "R"), (0, 0, "R"), (2, 2, "W"))),
           TaskEvent("NEG", (2,), ((3, 3, "R"), (1, 1, "W"))),
           DropRef(3), Flush()]
    out["edge_nan_inf"] = ev
    return out


def main():
    bench = []
    for name, events in edge_streams().items():
        for cfg in ("fused", "unfused", "w2"):
            bench.append(case_from_events(name, events, cfg))
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
