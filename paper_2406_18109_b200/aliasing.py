"""Aliased views of one store inside a single launch point.

The reference binds every argument of a point to a numpy view of the whole
store (``_region``, executor.py:119-121) and evaluates the kernel statement by
statement over whole arrays (``interpret``, kernels.py:749-765).  A task may
therefore read and write one store through two arguments -- ``ir.py:176-190``
only rejects duplicate *effectful* arguments -- and numpy gives it a precise
meaning: the right-hand side of a statement is computed into a fresh array
before it is assigned, and a statement sees every earlier statement's stores.

The device kernel runs one thread per element pair with the loads of a pair
hoisted, so two views of one store need care:

* identical rects: element ``i`` of both views is the same address and only
  the thread that owns ``i`` touches it.  Loads that follow a store to the
  alias in statement order must see the stored value; the kernel is rewritten
  so that every access of the alias group goes through one slot, whose
  store-to-load order the JIT already honours (``rewrite``).
* overlapping but different rects: another thread may write the element this
  thread reads.  If every read of the view happens in or before the first
  statement that writes the store (numpy's read-then-assign semantics), the
  view is copied to scratch before the launch and the kernel reads the copy
  (``copy_in`` slots).  Anything else -- reads after an overlapping write, or
  per-element nests with offsets (kernels.py:766-783, sequential numpy
  semantics) -- raises ``UnsupportedError`` instead of racing.
"""

from __future__ import annotations

from . import regions as rg
from .errors import UnsupportedError
from .ir import KProg, Slot, stmt_expr

_WRITE_PRIVS = (None, "W", "RW")


def _positions(kp: KProg):
    """Per slot: positions (nest, stmt) of its loads, stores and reductions."""
    loads: dict[int, list] = {}
    stores: dict[int, list] = {}
    reduces: dict[int, list] = {}
    offsets: set[int] = set()
    for n, (_dom, _rank, stmts) in enumerate(kp.nests):
        for k, st in enumerate(stmts):
            for slot, offs in _expr_loads(stmt_expr(st)):
                loads.setdefault(slot, []).append((n, k))
                if offs and any(offs):
                    offsets.add(slot)
            if st[0] == "store":
                stores.setdefault(st[1], []).append((n, k))
                if any(st[2]):
                    offsets.add(st[1])
            elif st[0] == "reduce":
                reduces.setdefault(st[1], []).append((n, k))
    return loads, stores, reduces, offsets


def _expr_loads(e: tuple):
    tag = e[0]
    if tag == "ld":
        yield (e[1], e[2])
    elif tag == "bin":
        yield from _expr_loads(e[2])
        yield from _expr_loads(e[3])
    elif tag == "neg":
        yield from _expr_loads(e[1])
    elif tag == "sel":
        for x in e[1:]:
            yield from _expr_loads(x)


def plan(kp: KProg, store_of_slot: dict[int, int], rects: dict[int, tuple]):
    """Classify the aliasing of one point's bound views.

    ``store_of_slot`` / ``rects``: store id and bound rect of every non-local
    slot.  Returns ``(mapping, copy_in)``: a slot renaming for identical-rect
    groups that contain a stored slot (None when there is none) and the slots
    to be read from a scratch copy.  Raises ``UnsupportedError`` for patterns
    whose numpy semantics the device kernel cannot reproduce.
    """
    loads, stores, reduces, offsets = _positions(kp)
    by_store: dict[int, list[int]] = {}
    for s, sid in store_of_slot.items():
        by_store.setdefault(sid, []).append(s)
    mapping: dict[int, int] = {}
    copy_in: list[int] = []
    for sid, slots in by_store.items():
        if len(slots) < 2:
            continue
        written = [s for s in slots if s in stores]
        if not written:
            continue
        nonempty = [s for s in slots if not rg.empty(rects[s])]
        for w in written:
            if rg.empty(rects[w]):
                continue
            for r in nonempty:
                if r == w or not rg.overlaps(rects[r], rects[w]):
                    continue
                if r in offsets or w in offsets:
                    raise UnsupportedError(
                        f"{kp.slots[w].name} and {kp.slots[r].name} view store {sid} with overlap inside a "
                        "per-element nest (sequential numpy semantics)")
                if r in reduces or w in reduces:
                    raise UnsupportedError(
                        f"{kp.slots[r].name}: a reduction target aliases a stored view of store {sid}")
                if rects[r] == rects[w]:
                    continue  # handled by the identical-rect rewrite below
                if r in stores:
                    raise UnsupportedError(
                        f"{kp.slots[w].name} and {kp.slots[r].name} write overlapping, different rects of store {sid}")
                first_w = min(stores[w])
                if any(pos > first_w for pos in loads.get(r, ())):
                    raise UnsupportedError(
                        f"{kp.slots[r].name} reads store {sid} after an overlapping write through {kp.slots[w].name}")
                if r not in copy_in:
                    copy_in.append(r)
        # identical-rect groups with a stored member: one slot for all accesses
        groups: list[list[int]] = []
        for s in sorted(nonempty):
            for g in groups:
                if rects[g[0]] == rects[s]:
                    g.append(s)
                    break
            else:
                groups.append([s])
        for g in groups:
            if len(g) < 2 or not any(s in stores for s in g):
                continue
            if any(s in copy_in for s in g):
                raise UnsupportedError(f"store {sid}: a view is both copied in and aliased")
            if any(kp.slots[s].priv not in _WRITE_PRIVS for s in g if s in stores):
                continue  # a store into a read-only view: let the JIT raise PrivilegeError
            canon = min(s for s in g if s in stores)
            for s in g:
                if s != canon:
                    mapping[s] = canon
    return (mapping or None), copy_in


def _rw_expr(e: tuple, m: dict[int, int]) -> tuple:
    tag = e[0]
    if tag == "ld":
        return ("ld", m.get(e[1], e[1]), e[2])
    if tag == "bin":
        return ("bin", e[1], _rw_expr(e[2], m), _rw_expr(e[3], m))
    if tag == "neg":
        return ("neg", _rw_expr(e[1], m))
    if tag == "sel":
        return ("sel", _rw_expr(e[1], m), _rw_expr(e[2], m), _rw_expr(e[3], m))
    return e


def rewrite(kp: KProg, mapping: dict[int, int]) -> KProg:
    """Route every load/store of an aliased slot through its group's canonical slot.

    The canonical slot keeps a write privilege; the other members stay bound
    (same view) but are no longer referenced."""
    nests = []
    for dom, rank, stmts in kp.nests:
        out = []
        for st in stmts:
            if st[0] == "set":
                out.append(("set", st[1], _rw_expr(st[2], mapping)))
            elif st[0] == "store":
                out.append(("store", mapping.get(st[1], st[1]), st[2], _rw_expr(st[3], mapping)))
            else:
                out.append(("reduce", st[1], _rw_expr(st[2], mapping)))
        nests.append((mapping.get(dom, dom), rank, tuple(out)))
    slots = list(kp.slots)
    for s, c in mapping.items():
        if slots[c].priv == "W" and kp.slots[s].priv in ("R", "RW"):
            slots[c] = Slot(slots[c].name, slots[c].arg, slots[c].local, "RW", slots[c].decl_rank)
    return KProg(tuple(slots), kp.scalar_names, kp.ntemps, tuple(nests), kp.fused_names)


_COPY: dict[int, KProg] = {}


def copy_kprog(rank: int) -> KProg:
    """``dst = src`` over a rank-``rank`` view (the copy-in kernel)."""
    kp = _COPY.get(rank)
    if kp is None:
        z = (0,) * rank
        kp = KProg((Slot("c0", 0, False, "R", rank), Slot("c1", 1, False, "W", rank)), (), 0,
                   ((1, rank, (("store", 1, z, ("ld", 0, z)),)),), False)
        _COPY[rank] = kp
    return kp
