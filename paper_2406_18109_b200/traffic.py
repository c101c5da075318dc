"""Algorithmic (compulsory) HBM bytes of a launch -- the roofline numerator.

SURVEY §8(d): each non-temporary store region a launch point touches is read
once and/or written once; RW counts both; temporaries count 0 (they live in
registers); rank-0 stores and halo bytes are ignored.  Aliased views of one
store (the stencil's five views of ``grid``) count their union once.  The
reference's own figure, ``count_memory_traffic`` (kernels.py:625-640), counts
every Load separately and so double-counts aliased views; it is reported
beside this one, not used as the denominator.

``SPMV_CSR`` reads x through a replicated view, but only the columns its
rows reference are compulsory: for the banded Poisson tiles that is the
tile's own rows plus one grid row on either side.
"""

from __future__ import annotations

from typing import Iterable

from . import regions as rg
from .initheap import poisson_tile_layout
from .ir import KProg, TaskDesc, hbm_reads, rect_of


def launch_bytes(task: TaskDesc, kp: KProg | None, temp_positions: Iterable[int], shapes, dtypes,
                 points: Iterable[int] | None = None, init: dict | None = None) -> int:
    temp_positions = frozenset(temp_positions)
    pts = list(task.points())
    sel = range(len(pts)) if points is None else points
    if kp is None:
        rd = [a.reads or a.reduces or (a.writes and task.kind == "OPAQUE") for a in task.args]
        wr = [a.writes for a in task.args]
    else:
        stored = {st[1] for _, _, sts in kp.nests for st in sts if st[0] == "store"}
        loaded = hbm_reads(kp)
        rd = [False] * len(task.args)
        wr = [False] * len(task.args)
        for i, s in enumerate(kp.slots):
            if s.local:
                continue
            a = task.args[s.arg]
            rd[s.arg] = rd[s.arg] or i in loaded
            wr[s.arg] = wr[s.arg] or (i in stored and a.writes)
    total = 0
    for i in sel:
        p = pts[i]
        reads: dict[int, list] = {}
        writes: dict[int, list] = {}
        for j, a in enumerate(task.args):
            if j in temp_positions or not shapes[a.store]:
                continue
            rect = rect_of(shapes[a.store], a.part, p)
            if task.kind == "SPMV_CSR" and j == 3 and init is not None:
                rect = _csr_x_footprint(task, p, shapes, init)
            if rd[j]:
                reads[a.store] = rg.add(reads.get(a.store, []), rect)
            if wr[j]:
                writes[a.store] = rg.add(writes.get(a.store, []), rect)
        for sid, rects in reads.items():
            es = 4 if dtypes.get(sid) == "i32" else 8
            total += es * sum(rg.volume(r) for r in rects)
        for sid, rects in writes.items():
            es = 4 if dtypes.get(sid) == "i32" else 8
            total += es * sum(rg.volume(r) for r in rects)
    return total


def _csr_x_footprint(task: TaskDesc, p, shapes, init):
    spec = init.get(task.args[0].store)
    n = shapes[task.args[3].store][0]
    if not spec or "nx" not in spec:
        return ((0,), (n,))
    lay = poisson_tile_layout(int(spec["nx"]), int(spec["ny"]), int(spec["k"]))
    t, nx = lay["t"], lay["nx"]
    q = p[0]
    return ((max(0, q * t - nx),), (min(n, (q + 1) * t + nx),))


def reference_traffic(kp: KProg, task: TaskDesc, temp_positions, shapes) -> int:
    """count_memory_traffic x 8 bytes (kernels.py:625-640 with pipeline.py:347-369 scaling)."""
    p0 = tuple(0 for _ in task.launch)
    ext = {}
    for i, s in enumerate(kp.slots):
        a = task.args[s.arg]
        lo, hi = rect_of(shapes[a.store], a.part, p0)
        ext[i] = tuple(max(0, h - l) for l, h in zip(lo, hi))
    loads = stores = 0
    for dom, _, sts in kp.nests:
        vol = 1
        for e in ext[dom]:
            vol *= e
        for st in sts:
            e = st[3] if st[0] == "store" else st[2]
            loads += _nloads(e) * vol
            if st[0] in ("store", "reduce"):
                stores += vol
    return 8 * (loads + stores) * task.volume


def _nloads(e) -> int:
    tag = e[0]
    if tag == "ld":
        return 1
    if tag == "bin":
        return _nloads(e[2]) + _nloads(e[3])
    if tag == "neg":
        return _nloads(e[1])
    if tag == "sel":
        return _nloads(e[1]) + _nloads(e[2]) + _nloads(e[3])
    return 0
