"""Backend-side descriptions of what a fused window hands the executor.

The reference front end (``diffusekit``) produces frozen dataclasses: an
``IndexTask`` (``ir.py:172-190``) and an optimized ``Kernel``
(``kernels.py:134-151``).  The B200 backend never executes those objects
directly.  It lowers them once into two plain, hashable forms:

* :class:`TaskDesc` -- launch extents, per-argument (store, partition,
  privilege) and positional scalar values.  Partitions become
  :class:`PartDesc` tuples; ``rect_of`` restates ``sub_store_bounds``
  (``ir.py:249-267``) on them.
* :class:`KProg` -- the kernel with buffer names resolved to *slots*, scalar
  names resolved to positions and temporaries numbered.  Expressions are
  nested tuples.  ``KProg.wire()`` is the text handed to the C++ JIT
  (``dk_kernel_compile``).

Lowering is duck-typed on the reference class names so the same code accepts
the reference's objects (drop-in use inside ``GpuSession``) and the JSON form
recorded by ``tools/capture_plans.py`` (plan replay on the GPU box, where the
reference is not installed).
"""

from __future__ import annotations

import itertools
import struct
from dataclasses import dataclass, field
from typing import Any, Iterator, Sequence

PRIVS = ("R", "W", "Rd", "RW")
BIN_OPS = ("+", "-", "*", "/", "**", "min", "max", "lt", "le", "eq")


class IRError(ValueError):
    """A task or kernel cannot be lowered to the backend form."""


# --------------------------------------------------------------------------
# tasks
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class PartDesc:
    """``kind`` is "none" (replication) or "tiling" (affine tile, ir.py:116-129)."""

    kind: str
    tile: tuple[int, ...] = ()
    offset: tuple[int, ...] = ()
    A: tuple[tuple[int, ...], ...] = ()
    b: tuple[int, ...] = ()

    @property
    def is_none(self) -> bool:
        return self.kind == "none"

    def project(self, p: Sequence[int]) -> tuple[int, ...]:
        return tuple(sum(a * c for a, c in zip(row, p)) + o for row, o in zip(self.A, self.b))


NONE_PART = PartDesc("none")


@dataclass(frozen=True)
class ArgDesc:
    store: int
    part: PartDesc
    priv: str  # one of PRIVS

    @property
    def reads(self) -> bool:
        return self.priv in ("R", "RW")

    @property
    def writes(self) -> bool:
        return self.priv in ("W", "RW")

    @property
    def reduces(self) -> bool:
        return self.priv == "Rd"


@dataclass(frozen=True)
class TaskDesc:
    kind: str
    launch: tuple[int, ...]
    args: tuple[ArgDesc, ...]
    scalars: tuple[float, ...] = ()
    scalar_names: tuple[str, ...] = ()

    def points(self) -> Iterator[tuple[int, ...]]:
        """Launch points in lexicographic order (ir.py:46-48)."""
        return itertools.product(*(range(e) for e in self.launch))

    def __hash__(self) -> int:  # cached: fused tasks carry dozens of arguments
        h = self.__dict__.get("_hash")
        if h is None:
            h = hash((self.kind, self.launch, self.args, self.scalars, self.scalar_names))
            object.__setattr__(self, "_hash", h)
        return h

    @property
    def volume(self) -> int:
        v = 1
        for e in self.launch:
            v *= e
        return v


Rect = tuple[tuple[int, ...], tuple[int, ...]]  # (lo, hi), half-open


def rect_of(shape: Sequence[int], part: PartDesc, p: Sequence[int]) -> Rect:
    """Clamped bounding box of ``part`` at launch point ``p`` (ir.py:249-267)."""
    if part.is_none:
        return (tuple(0 for _ in shape), tuple(shape))
    if len(part.A) != len(shape):
        raise IRError(f"partition of rank {len(part.A)} applied to a rank-{len(shape)} store")
    q0 = part.project(p)
    q1 = part.project([c + 1 for c in p])
    lo = [a * t + o for a, t, o in zip(q0, part.tile, part.offset)]
    hi = [a * t + o for a, t, o in zip(q1, part.tile, part.offset)]
    lo = tuple(min(max(v, 0), s) for v, s in zip(lo, shape))
    hi = tuple(min(max(v, 0), s) for v, s in zip(hi, shape))
    return (lo, hi)


def rect_extents(r: Rect) -> tuple[int, ...]:
    return tuple(max(0, h - l) for l, h in zip(*r))


def rect_volume(r: Rect) -> int:
    v = 1
    for e in rect_extents(r):
        v *= e
    return v


def _part_from_ref(part: Any) -> PartDesc:
    if hasattr(part, "tile"):
        return PartDesc(
            "tiling",
            tuple(int(v) for v in part.tile),
            tuple(int(v) for v in part.offset),
            tuple(tuple(int(v) for v in row) for row in part.proj.matrix),
            tuple(int(v) for v in part.proj.offset),
        )
    return NONE_PART


_PART_CACHE: dict[Any, PartDesc] = {}


def _part_cached(part: Any) -> PartDesc:
    # reference partitions are frozen (hash/eq by value); a fused window lowers
    # dozens of identical tilings every iteration
    try:
        hit = _PART_CACHE.get(part)
    except TypeError:
        return _part_from_ref(part)
    if hit is None:
        if len(_PART_CACHE) > 100_000:
            _PART_CACHE.clear()
        hit = _PART_CACHE[part] = _part_from_ref(part)
    return hit


def lower_task(task: Any) -> TaskDesc:
    """Reference ``IndexTask`` (ir.py:172-190) -> :class:`TaskDesc`."""
    if isinstance(task, TaskDesc):
        return task
    args = tuple(
        ArgDesc(int(a.store), _part_cached(a.partition), a.privilege.value) for a in task.args
    )
    return TaskDesc(
        task.kind,
        tuple(int(e) for e in task.domain.extents),
        args,
        tuple(float(v) for _, v in task.scalars),
        tuple(str(n) for n, _ in task.scalars),
    )


# --------------------------------------------------------------------------
# kernels
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Slot:
    """One buffer of the kernel: a heap-bound parameter or a task-local buffer."""

    name: str
    arg: int  # fused / plain argument position the buffer binds to
    local: bool
    priv: str | None  # None for locals
    decl_rank: int


@dataclass(frozen=True)
class KProg:
    """A kernel in slot form.

    ``nests`` is a tuple of ``(domain_slot, rank, stmts)``; statements are
    ``("set", t, e)``, ``("store", slot, offsets, e)`` and ``("reduce", slot, e)``;
    expressions are ``("ld", slot, offsets)``, ``("sc", i)``, ``("c", value)``,
    ``("t", i)``, ``("bin", op, l, r)``, ``("neg", x)`` and ``("sel", c, t, f)``.
    """

    slots: tuple[Slot, ...]
    scalar_names: tuple[str, ...]
    ntemps: int
    nests: tuple
    fused_names: bool
    text: str = field(default="", compare=False)

    def slot_index(self, name: str) -> int:
        for i, s in enumerate(self.slots):
            if s.name == name:
                return i
        raise IRError(f"kernel has no buffer {name!r}")

    def wire(self, ranks: Sequence[int]) -> str:
        """Text program for the C++ JIT, specialised on actual bound ranks."""
        out = [f"DK1 {len(self.slots)} {len(self.scalar_names)} {self.ntemps} {len(self.nests)}"]
        for i, s in enumerate(self.slots):
            out.append(f"slot {i} {ranks[i]} {'L' if s.local else 'P'} {s.priv or '-'}")
        for dom, rank, stmts in self.nests:
            out.append(f"nest {dom} {rank} {len(stmts)}")
            for st in stmts:
                if st[0] == "set":
                    out.append(f" T {st[1]} {_wire_expr(st[2])}")
                elif st[0] == "store":
                    offs = ",".join(str(o) for o in st[2]) or "-"
                    out.append(f" S {st[1]} {offs} {_wire_expr(st[3])}")
                else:
                    out.append(f" A {st[1]} {_wire_expr(st[2])}")
        out.append("end")
        return "\n".join(out) + "\n"


def _wire_expr(e: tuple) -> str:
    tag = e[0]
    if tag == "ld":
        offs = ",".join(str(o) for o in e[2]) or "-"
        return f"(L {e[1]} {offs})"
    if tag == "sc":
        return f"(P {e[1]})"
    if tag == "c":
        return f"(C {struct.unpack('<Q', struct.pack('<d', e[1]))[0]:016x})"
    if tag == "t":
        return f"(V {e[1]})"
    if tag == "bin":
        return f"(B {e[1]} {_wire_expr(e[2])} {_wire_expr(e[3])})"
    if tag == "neg":
        return f"(N {_wire_expr(e[1])})"
    return f"(Q {_wire_expr(e[1])} {_wire_expr(e[2])} {_wire_expr(e[3])})"


def _slot_arg(name: str) -> int:
    if len(name) < 2 or name[0] not in "abl" or not name[1:].isdigit():
        raise IRError(f"buffer name {name!r} is not a{{j}}/b{{j}}/l{{j}}")
    return int(name[1:])


class _Lowerer:
    def __init__(self, slot_of: dict[str, int], scal_of: dict[str, int]) -> None:
        self.slot_of = slot_of
        self.scal_of = scal_of
        self.temp_of: dict[str, int] = {}

    def expr(self, e: Any) -> tuple:
        cls = type(e).__name__
        if cls == "Load":
            if e.buf not in self.slot_of:
                raise IRError(f"load of unknown buffer {e.buf!r}")
            return ("ld", self.slot_of[e.buf], tuple(int(o) for o in e.offsets))
        if cls == "ScalarRef":
            if e.name not in self.scal_of:
                raise IRError(f"unknown scalar {e.name!r}")
            return ("sc", self.scal_of[e.name])
        if cls == "Const":
            return ("c", float(e.value))
        if cls == "TempRef":
            if e.name not in self.temp_of:
                raise IRError(f"temporary {e.name!r} read before it is set")
            return ("t", self.temp_of[e.name])
        if cls == "Bin":
            if e.op not in BIN_OPS:
                raise IRError(f"unknown binary op {e.op!r}")
            return ("bin", e.op, self.expr(e.lhs), self.expr(e.rhs))
        if cls == "Un":
            if e.op != "neg":
                raise IRError(f"unknown unary op {e.op!r}")
            return ("neg", self.expr(e.x))
        if cls == "Select":
            return ("sel", self.expr(e.cond), self.expr(e.if_true), self.expr(e.if_false))
        raise IRError(f"unknown expression node {cls}")

    def stmt(self, s: Any) -> tuple:
        cls = type(s).__name__
        if cls == "SetTemp":
            e = self.expr(s.expr)
            t = self.temp_of.setdefault(s.name, len(self.temp_of))
            return ("set", t, e)
        if cls == "StoreStmt":
            return ("store", self.slot_of[s.buf], tuple(int(o) for o in s.offsets), self.expr(s.expr))
        if cls == "ReduceStmt":
            return ("reduce", self.slot_of[s.buf], self.expr(s.expr))
        raise IRError(f"unknown statement node {cls}")


def lower_kernel(kernel: Any, fused_names: bool) -> KProg:
    """Reference ``Kernel`` (kernels.py:134-151) -> :class:`KProg`."""
    if isinstance(kernel, KProg):
        return kernel
    slots: list[Slot] = []
    for p in kernel.buf_params:
        slots.append(Slot(p.name, _slot_arg(p.name), False, p.privilege.value, int(p.rank)))
    for l in kernel.locals:
        slots.append(Slot(l.name, _slot_arg(l.name), True, None, int(l.rank)))
    slot_of = {s.name: i for i, s in enumerate(slots)}
    scal_of = {sp.name: i for i, sp in enumerate(kernel.scalar_params)}
    low = _Lowerer(slot_of, scal_of)
    nests = []
    for nest in kernel.nests:
        if nest.domain not in slot_of:
            raise IRError(f"nest iterates over unknown buffer {nest.domain!r}")
        nests.append((slot_of[nest.domain], int(nest.rank), tuple(low.stmt(s) for s in nest.body)))
    return KProg(
        tuple(slots),
        tuple(sp.name for sp in kernel.scalar_params),
        len(low.temp_of),
        tuple(nests),
        fused_names,
    )


def expr_slots(e: tuple) -> Iterator[tuple[int, tuple[int, ...]]]:
    """(slot, offsets) of every load in an expression."""
    tag = e[0]
    if tag == "ld":
        yield (e[1], e[2])
    elif tag == "bin":
        yield from expr_slots(e[2])
        yield from expr_slots(e[3])
    elif tag == "neg":
        yield from expr_slots(e[1])
    elif tag == "sel":
        yield from expr_slots(e[1])
        yield from expr_slots(e[2])
        yield from expr_slots(e[3])


def stmt_expr(st: tuple) -> tuple:
    return st[3] if st[0] == "store" else st[2]


def slot_access(kp: KProg) -> tuple[set[int], set[int], set[int]]:
    """(read_first, stored, reduced) slots of a kernel.

    ``read_first``: slots whose old contents the kernel observes -- a load that
    precedes (in nest, then statement order) every store to the slot.  A store
    covers its whole view (the JIT requires target extents == nest domain), so
    a slot written before it is read needs no prior contents: no HBM read, no
    initialisation, no transfer.  Loads in a later nest of a slot stored by an
    earlier nest read HBM but see this launch's own values, not older ones.
    """
    read_first: set[int] = set()
    stored: set[int] = set()
    reduced: set[int] = set()
    for _dom, _rank, stmts in kp.nests:
        for st in stmts:
            for slot, _offs in expr_slots(stmt_expr(st)):
                if slot not in stored:
                    read_first.add(slot)
            if st[0] == "store":
                stored.add(st[1])
            elif st[0] == "reduce":
                reduced.add(st[1])
    return read_first, stored, reduced


def hbm_reads(kp: KProg) -> set[int]:
    """Slots the kernel loads from HBM: per nest, loaded before stored in that nest."""
    out: set[int] = set()
    for _dom, _rank, stmts in kp.nests:
        stored_here: set[int] = set()
        for st in stmts:
            for slot, _offs in expr_slots(stmt_expr(st)):
                if slot not in stored_here:
                    out.add(slot)
            if st[0] == "store":
                stored_here.add(st[1])
    return out


# --------------------------------------------------------------------------
# JSON codec (plan traces recorded from the reference front end)
# --------------------------------------------------------------------------


def part_to_json(p: PartDesc) -> Any:
    if p.is_none:
        return "none"
    return {"tile": list(p.tile), "offset": list(p.offset), "A": [list(r) for r in p.A], "b": list(p.b)}


def part_from_json(o: Any) -> PartDesc:
    if o == "none":
        return NONE_PART
    return PartDesc(
        "tiling",
        tuple(o["tile"]),
        tuple(o["offset"]),
        tuple(tuple(r) for r in o["A"]),
        tuple(o["b"]),
    )


def task_to_json(t: TaskDesc) -> dict:
    return {
        "kind": t.kind,
        "launch": list(t.launch),
        "args": [[a.store, part_to_json(a.part), a.priv] for a in t.args],
        "scalars": [[n, v] for n, v in zip(t.scalar_names, t.scalars)],
    }


def task_from_json(o: dict) -> TaskDesc:
    sc = o.get("scalars", [])
    return TaskDesc(
        o["kind"],
        tuple(o["launch"]),
        tuple(ArgDesc(int(s), part_from_json(p), pr) for s, p, pr in o["args"]),
        tuple(float(v) for _, v in sc),
        tuple(str(n) for n, _ in sc),
    )


def _expr_to_json(e: tuple) -> list:
    tag = e[0]
    if tag == "ld":
        return ["ld", e[1], list(e[2])]
    if tag in ("sc", "t"):
        return [tag, e[1]]
    if tag == "c":
        return ["c", e[1].hex()]
    if tag == "bin":
        return ["bin", e[1], _expr_to_json(e[2]), _expr_to_json(e[3])]
    if tag == "neg":
        return ["neg", _expr_to_json(e[1])]
    return ["sel", _expr_to_json(e[1]), _expr_to_json(e[2]), _expr_to_json(e[3])]


def _expr_from_json(o: list) -> tuple:
    tag = o[0]
    if tag == "ld":
        return ("ld", int(o[1]), tuple(o[2]))
    if tag in ("sc", "t"):
        return (tag, int(o[1]))
    if tag == "c":
        return ("c", float.fromhex(o[1]))
    if tag == "bin":
        return ("bin", o[1], _expr_from_json(o[2]), _expr_from_json(o[3]))
    if tag == "neg":
        return ("neg", _expr_from_json(o[1]))
    return ("sel", _expr_from_json(o[1]), _expr_from_json(o[2]), _expr_from_json(o[3]))


def kprog_to_json(k: KProg) -> dict:
    nests = []
    for dom, rank, stmts in k.nests:
        js = []
        for st in stmts:
            if st[0] == "set":
                js.append(["set", st[1], _expr_to_json(st[2])])
            elif st[0] == "store":
                js.append(["store", st[1], list(st[2]), _expr_to_json(st[3])])
            else:
                js.append(["reduce", st[1], _expr_to_json(st[2])])
        nests.append([dom, rank, js])
    return {
        "slots": [[s.name, s.arg, s.local, s.priv, s.decl_rank] for s in k.slots],
        "scalars": list(k.scalar_names),
        "ntemps": k.ntemps,
        "nests": nests,
        "fused": k.fused_names,
        "text": k.text,
    }


def kprog_from_json(o: dict) -> KProg:
    nests = []
    for dom, rank, js in o["nests"]:
        stmts = []
        for st in js:
            if st[0] == "set":
                stmts.append(("set", int(st[1]), _expr_from_json(st[2])))
            elif st[0] == "store":
                stmts.append(("store", int(st[1]), tuple(st[2]), _expr_from_json(st[3])))
            else:
                stmts.append(("reduce", int(st[1]), _expr_from_json(st[2])))
        nests.append((int(dom), int(rank), tuple(stmts)))
    return KProg(
        tuple(Slot(n, int(a), bool(l), p, int(r)) for n, a, l, p, r in o["slots"]),
        tuple(o["scalars"]),
        int(o["ntemps"]),
        tuple(nests),
        bool(o["fused"]),
        o.get("text", ""),
    )
