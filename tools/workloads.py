"""Harness event streams for the BASELINE configurations (build container only).

Each generator returns ``(events, init, dtypes, builtins_needed)`` where
``events`` are the reference's own trace events (``diffusekit.trace``), fed
unchanged to the reference ``Session``.  Three streams are new (SURVEY H7,
§8 d): the reference's ``gen_stencil`` launches ``(nodes, nodes)`` and its
``gen_cg_like`` runs SPMV on launch ``(1,)``, neither of which maps to 2 or 8
GPUs.

* ``stencil_bands`` -- ``gen_stencil`` (trace.py:242-277) on row bands, launch
  ``(k, 1)``, plus the residual ``SUB(work, center -> diff)``,
  ``DOT(diff, diff -> res)`` before the COPY.
* ``cg_csr``        -- ``gen_cg_like`` (trace.py:352-404) with the opaque dense
  SPMV replaced by ``SPMV_CSR`` over per-tile CSR stores of the 2-D Poisson
  matrix, rank-0 reduction targets zero-initialised (C4).
* ``pcg_csr``       -- Jacobi-preconditioned CG: dense MULT by the inverse
  diagonal fused with the sparse-library reductions (C5).
"""

from __future__ import annotations

from refcapture import import_reference

dk = import_reference()
from diffusekit.trace import (  # noqa: E402
    CreatePartition,
    CreateStore,
    DropRef,
    Flush,
    TaskEvent,
    gen_blackscholes_chain,
)

from paper_2406_18109_b200.initheap import poisson_tile_layout  # noqa: E402


class _B:
    def __init__(self) -> None:
        self.events = []
        self.ns = 0
        self.np = 0
        self.init: dict[int, dict] = {}
        self.dtypes: dict[int, str] = {}

    def store(self, shape, init=None, dtype=None) -> int:
        sid = self.ns
        self.ns += 1
        self.events.append(CreateStore(sid, tuple(shape)))
        if init is not None:
            self.init[sid] = init
        if dtype is not None:
            self.dtypes[sid] = dtype
        return sid

    def none(self, s) -> int:
        pid = self.np
        self.np += 1
        self.events.append(CreatePartition(pid, s, "none"))
        return pid

    def tiling(self, s, tile, offset, A=None, b=None) -> int:
        pid = self.np
        self.np += 1
        r = len(tile)
        if A is None:
            A = tuple(tuple(1 if i == j else 0 for j in range(r)) for i in range(r))
            b = (0,) * r
        self.events.append(CreatePartition(pid, s, "tiling", tuple(tile), tuple(offset), (tuple(A), tuple(b))))
        return pid

    def task(self, kind, dom, args, scalars=()) -> None:
        self.events.append(TaskEvent(kind, tuple(dom), tuple(args), tuple(scalars)))

    def drop(self, s) -> None:
        self.events.append(DropRef(s))

    def flush(self) -> None:
        self.events.append(Flush())


def blackscholes(size: int, nodes: int, iters: int):
    return gen_blackscholes_chain(size=size, nodes=nodes, iters=iters), {}, {}


def stencil_bands(n: int, k: int, iters: int, residual: bool = True):
    """Row-band 5-point stencil on an (n*k) x n interior, one band per point."""
    b = _B()
    grid = b.store((n * k + 2, n + 2))
    work = b.store((n * k, n))
    tile = (n, n)
    p_center = b.tiling(grid, tile, (1, 1))
    p_north = b.tiling(grid, tile, (0, 1))
    p_east = b.tiling(grid, tile, (1, 2))
    p_west = b.tiling(grid, tile, (1, 0))
    p_south = b.tiling(grid, tile, (2, 1))
    p_work = b.tiling(work, tile, (0, 0))
    launch = (k, 1)
    for _ in range(iters):
        tmp = [b.store((n * k, n)) for _ in range(5 if residual else 4)]
        pt = [b.tiling(s, tile, (0, 0)) for s in tmp]
        t1, t2, t3, avg = tmp[:4]
        b.task("ADD", launch, [(grid, p_center, "R"), (grid, p_north, "R"), (t1, pt[0], "W")])
        b.task("ADD", launch, [(t1, pt[0], "R"), (grid, p_east, "R"), (t2, pt[1], "W")])
        b.drop(t1)
        b.task("ADD", launch, [(t2, pt[1], "R"), (grid, p_west, "R"), (t3, pt[2], "W")])
        b.drop(t2)
        b.task("ADD", launch, [(t3, pt[2], "R"), (grid, p_south, "R"), (avg, pt[3], "W")])
        b.drop(t3)
        b.task("MULT", launch, [(avg, pt[3], "R"), (work, p_work, "W")], [("s", 0.2)])
        b.drop(avg)
        if residual:
            diff = tmp[4]
            res = b.store((), init={"kind": "zeros"})
            n_res = b.none(res)
            b.task("SUB", launch, [(work, p_work, "R"), (grid, p_center, "R"), (diff, pt[4], "W")])
            b.task("DOT", launch, [(diff, pt[4], "R"), (diff, pt[4], "R"), (res, n_res, "Rd")])
            b.drop(diff)
        b.task("COPY", launch, [(work, p_work, "R"), (grid, p_center, "W")])
        b.flush()
    return b.events, b.init, b.dtypes


def _csr_stores(b: _B, nx: int, ny: int, k: int):
    lay = poisson_tile_layout(nx, ny, k)
    t, nnz = lay["t"], lay["nnz_max"]
    spec = {"nx": nx, "ny": ny, "k": k}
    # per-tile CSR, concatenated: tile p owns rowptr[p*(t+1):(p+1)*(t+1)] (local
    # offsets) and cols/vals[p*nnz:(p+1)*nnz] (global column ids)
    rowptr = b.store((k * (t + 1),), init={"kind": "csr_rowptr", **spec}, dtype="i32")
    cols = b.store((k * nnz,), init={"kind": "csr_cols", **spec}, dtype="i32")
    vals = b.store((k * nnz,), init={"kind": "csr_vals", **spec})
    p_rp = b.tiling(rowptr, (t + 1,), (0,))
    p_cl = b.tiling(cols, (nnz,), (0,))
    p_vl = b.tiling(vals, (nnz,), (0,))
    return lay, (rowptr, p_rp), (cols, p_cl), (vals, p_vl)


def cg_csr(nx: int, ny: int, k: int, iters: int):
    """``gen_cg_like`` with a CSR Poisson SpMV on row tiles; real CG numerics."""
    b = _B()
    lay, rp, cl, vl = _csr_stores(b, nx, ny, k)
    n, t = lay["n"], lay["t"]
    x = b.store((n,), init={"kind": "zeros"})
    r = b.store((n,), init={"kind": "uniform", "seed": 0, "key": 1000})
    p = b.store((n,), init={"kind": "uniform", "seed": 0, "key": 1000})
    q = b.store((n,), init={"kind": "zeros"})
    resid = b.store((n,), init={"kind": "zeros"})
    n_p = b.none(p)
    p_x, p_r, p_p, p_q, p_res = (b.tiling(s, (t,), (0,)) for s in (x, r, p, q, resid))
    launch = (k,)
    for _ in range(iters):
        pq = b.store((), init={"kind": "zeros"})
        rs_old = b.store((), init={"kind": "zeros"})
        rs_new = b.store((), init={"kind": "zeros"})
        n_pq, n_rso, n_rsn = b.none(pq), b.none(rs_old), b.none(rs_new)
        w = [b.store((n,)) for _ in range(4)]
        pw = [b.tiling(s, (t,), (0,)) for s in w]
        b.task("SPMV_CSR", launch, [(rp[0], rp[1], "R"), (cl[0], cl[1], "R"), (vl[0], vl[1], "R"), (p, n_p, "R"), (q, p_q, "W")])
        b.task("DOT", launch, [(p, p_p, "R"), (q, p_q, "R"), (pq, n_pq, "Rd")])
        b.task("DOT", launch, [(r, p_r, "R"), (r, p_r, "R"), (rs_old, n_rso, "Rd")])
        b.task("AXPY_RATIO", launch, [(p, p_p, "R"), (x, p_x, "RW"), (rs_old, n_rso, "R"), (pq, n_pq, "R")])
        b.task("AXMY_RATIO", launch, [(q, p_q, "R"), (r, p_r, "RW"), (rs_old, n_rso, "R"), (pq, n_pq, "R")])
        b.drop(pq)
        b.task("DOT", launch, [(r, p_r, "R"), (r, p_r, "R"), (rs_new, n_rsn, "Rd")])
        b.task("XPBY_RATIO", launch, [(r, p_r, "R"), (p, p_p, "RW"), (rs_new, n_rsn, "R"), (rs_old, n_rso, "R")])
        b.drop(rs_old)  # rs_new stays live: it is the residual history
        b.task("COPY", launch, [(r, p_r, "R"), (w[0], pw[0], "W")])
        b.task("NEG", launch, [(w[0], pw[0], "R"), (w[1], pw[1], "W")])
        b.drop(w[0])
        b.task("MULT", launch, [(w[1], pw[1], "R"), (w[2], pw[2], "W")], [("s", 2.0)])
        b.drop(w[1])
        b.task("ADD", launch, [(w[2], pw[2], "R"), (r, p_r, "R"), (w[3], pw[3], "W")])
        b.drop(w[2])
        b.task("COPY", launch, [(w[3], pw[3], "R"), (resid, p_res, "W")])
        b.drop(w[3])
        b.flush()
    return b.events, b.init, b.dtypes


def pcg_csr(nx: int, ny: int, k: int, iters: int):
    """Jacobi-preconditioned CG: dense MULT(r, invdiag) fused with sparse-path reductions."""
    b = _B()
    lay, rp, cl, vl = _csr_stores(b, nx, ny, k)
    n, t = lay["n"], lay["t"]
    x = b.store((n,), init={"kind": "zeros"})
    r = b.store((n,), init={"kind": "uniform", "seed": 0, "key": 1000})
    invd = b.store((n,), init={"kind": "poisson_invdiag"})
    # z0 = invdiag * r0 = r0 / 4 exactly; p0 = z0
    z = b.store((n,), init={"kind": "uniform", "seed": 0, "key": 1000, "scale": 0.25})
    p = b.store((n,), init={"kind": "uniform", "seed": 0, "key": 1000, "scale": 0.25})
    q = b.store((n,), init={"kind": "zeros"})
    n_p = b.none(p)
    p_x, p_r, p_d, p_z, p_p, p_q = (b.tiling(s, (t,), (0,)) for s in (x, r, invd, z, p, q))
    launch = (k,)
    for _ in range(iters):
        pq = b.store((), init={"kind": "zeros"})
        rz_old = b.store((), init={"kind": "zeros"})
        rz_new = b.store((), init={"kind": "zeros"})
        n_pq, n_old, n_new = b.none(pq), b.none(rz_old), b.none(rz_new)
        b.task("SPMV_CSR", launch, [(rp[0], rp[1], "R"), (cl[0], cl[1], "R"), (vl[0], vl[1], "R"), (p, n_p, "R"), (q, p_q, "W")])
        b.task("DOT", launch, [(p, p_p, "R"), (q, p_q, "R"), (pq, n_pq, "Rd")])
        b.task("DOT", launch, [(r, p_r, "R"), (z, p_z, "R"), (rz_old, n_old, "Rd")])
        b.task("AXPY_RATIO", launch, [(p, p_p, "R"), (x, p_x, "RW"), (rz_old, n_old, "R"), (pq, n_pq, "R")])
        b.task("AXMY_RATIO", launch, [(q, p_q, "R"), (r, p_r, "RW"), (rz_old, n_old, "R"), (pq, n_pq, "R")])
        b.drop(pq)
        b.task("MULT", launch, [(r, p_r, "R"), (invd, p_d, "R"), (z, p_z, "W")])
        b.task("DOT", launch, [(r, p_r, "R"), (z, p_z, "R"), (rz_new, n_new, "Rd")])
        b.task("XPBY_RATIO", launch, [(z, p_z, "R"), (p, p_p, "RW"), (rz_new, n_new, "R"), (rz_old, n_old, "R")])
        b.drop(rz_old)
        b.flush()
    return b.events, b.init, b.dtypes


# --------------------------------------------------------------------------
# JSON-lines: the reference's own trace format (trace.py:73-192)
# --------------------------------------------------------------------------
# The new workloads are written with the reference's printer and read with its
# parser, so ``diffusekit analyze / canon / run`` inspect them unchanged.  Their
# initial contents (zero reduction targets, CSR tiles, seeded uniform vectors)
# and backend dtype overrides travel as extra keys on the ``create_store`` line
# ("init", "dtype"): the reference parser reads only the keys it knows
# (trace.py:128-137), so the file stays a valid reference trace.


def write_jsonl(events, init=None, dtypes=None) -> str:
    import json

    from diffusekit.trace import CreateStore, event_to_json

    init, dtypes = dict(init or {}), dict(dtypes or {})
    lines = []
    for ev in events:
        obj = event_to_json(ev)
        if isinstance(ev, CreateStore):
            if ev.id in init:
                obj["init"] = init[ev.id]
            if ev.id in dtypes:
                obj["dtype"] = dtypes[ev.id]
        lines.append(json.dumps(obj))
    return "\n".join(lines) + "\n"


def read_jsonl(text: str):
    """(events, init, dtypes): the reference parser's events plus the harness annotations."""
    import json

    from diffusekit.trace import parse_trace

    events = parse_trace(text)
    init, dtypes = {}, {}
    for raw in text.splitlines():
        raw = raw.strip()
        if not raw:
            continue
        obj = json.loads(raw)
        if obj.get("event") == "create_store":
            if "init" in obj:
                init[int(obj["id"])] = obj["init"]
            if "dtype" in obj:
                dtypes[int(obj["id"])] = obj["dtype"]
    return events, init, dtypes


def cli_main():
    """python tools/workloads.py {stencil|cg|pcg|bs} [size args] > trace.jsonl"""
    import sys

    kind, *a = sys.argv[1:]
    a = [int(v) for v in a]
    gen = {"stencil": stencil_bands, "cg": cg_csr, "pcg": pcg_csr, "bs": blackscholes}[kind]
    out = gen(*a)
    events, init, dtypes = (out + ({},))[:3] if len(out) == 2 else out
    sys.stdout.write(write_jsonl(events, init, dtypes))


if __name__ == "__main__":
    cli_main()
