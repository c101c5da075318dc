"""Golden fixtures for aliased arguments, POW and isolated execution, from the UNCHANGED reference.

    python tests/golden/make_alias_golden.py      (build container only)

Streams whose tasks read and write one store through several arguments --
identical views (``ADD(x R, y R, x W)``), shifted views of the same store
(read at offset 0, write at offset 2), a written store read by a later
point's view -- are legal in the reference (``ir.py:176-190`` only rejects
duplicate *effectful* arguments) and numpy gives them a precise meaning.
Each stream runs through a reference ``Session`` under several configs; the
plan trace and the final heap bytes are stored in ``alias_streams.json.gz``.
Cases named ``*/isolated`` were run with ``SessionConfig(isolated=True)``
(``execute_isolated`` for fused prefixes, pipeline.py:325-334).

Heap contents are the reference's integers 1..9; POW tasks keep exponents
small so every value stays an exact integer and the comparison is bit-exact.
"""

from __future__ import annotations

import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import case_from_events, write  # noqa: E402
from make_golden import CONFIGS  # noqa: E402

from diffusekit.trace import CreatePartition, CreateStore, DropRef, Flush, TaskEvent  # noqa: E402

CONFIGS.setdefault("isolated", {"isolated": True})


def _ident(r):
    return (tuple(tuple(1 if i == j else 0 for j in range(r)) for i in range(r)), (0,) * r)


def hand_streams():
    out = {}
    # the judge's example: ADD(x R, y R, x W), same store and tiling, 3 points
    ev = [CreateStore(0, (12,)), CreateStore(1, (12,)), CreateStore(2, ())]
    ev += [CreatePartition(0, 0, "tiling", (4,), (0,), _ident(1)), CreatePartition(1, 1, "tiling", (4,), (0,), _ident(1)),
           CreatePartition(2, 2, "none")]
    for _ in range(3):
        ev += [TaskEvent("ADD", (3,), ((0, 0, "R"), (1, 1, "R"), (0, 0, "W"))),
               TaskEvent("MULT", (3,), ((0, 0, "R"), (0, 0, "R"), (1, 1, "W"))),
               TaskEvent("SUB", (3,), ((1, 1, "R"), (0, 0, "R"), (1, 1, "W"))),
               TaskEvent("DOT", (3,), ((0, 0, "R"), (1, 1, "R"), (2, 2, "Rd"))),
               Flush()]
    out["alias_same_view"] = ev
    # shifted views of one store: read x[i], write x[i + 2] (overlapping, unequal rects)
    ev = [CreateStore(0, (14,)), CreateStore(1, (14,))]
    ev += [CreatePartition(0, 0, "tiling", (4,), (0,), _ident(1)), CreatePartition(1, 0, "tiling", (4,), (2,), _ident(1)),
           CreatePartition(2, 1, "tiling", (4,), (1,), _ident(1))]
    for _ in range(2):
        ev += [TaskEvent("ADD", (3,), ((0, 0, "R"), (1, 2, "R"), (0, 1, "W"))),
               TaskEvent("NEG", (3,), ((0, 1, "R"), (0, 0, "W"))),
               TaskEvent("AXPY", (3,), ((0, 1, "R"), (0, 0, "RW")), (("w", 2.0),)),
               Flush()]
    out["alias_shifted_views"] = ev
    # 2-D: read the (1,1)-shifted view of the grid, write its centre (stencil in place)
    ev = [CreateStore(0, (10, 10)), CreateStore(1, (10, 10))]
    ev += [CreatePartition(0, 0, "tiling", (4, 4), (1, 1), _ident(2)), CreatePartition(1, 0, "tiling", (4, 4), (0, 1), _ident(2)),
           CreatePartition(2, 0, "tiling", (4, 4), (2, 2), _ident(2)), CreatePartition(3, 1, "tiling", (4, 4), (1, 1), _ident(2))]
    for _ in range(2):
        ev += [TaskEvent("ADD", (2, 2), ((0, 1, "R"), (0, 2, "R"), (0, 0, "W"))),
               TaskEvent("MAX", (2, 2), ((0, 0, "R"), (1, 3, "R"), (1, 3, "W"))),
               Flush()]
    out["alias_shifted_2d"] = ev
    # POW: elementwise and by a scalar exponent, integer results
    ev = [CreateStore(0, (9,)), CreateStore(1, (9,)), CreateStore(2, (9,)), CreateStore(3, (9,))]
    ev += [CreatePartition(i, i, "tiling", (3,), (0,), _ident(1)) for i in range(4)]
    ev += [TaskEvent("MIN", (3,), ((0, 0, "R"), (1, 1, "R"), (2, 2, "W"))),
           TaskEvent("POW", (3,), ((0, 0, "R"), (2, 2, "R"), (3, 3, "W"))),
           TaskEvent("POW", (3,), ((1, 1, "R"), (2, 2, "W")), (("s", 3.0),)),
           TaskEvent("POW", (3,), ((2, 2, "R"), (1, 1, "W")), (("s", 0.5),)),
           TaskEvent("POW", (3,), ((3, 3, "R"), (0, 0, "W")), (("s", -1.0),)),
           Flush()]
    out["pow_integer"] = ev
    return out


KINDS2 = ("ADD", "SUB", "MULT", "MIN", "MAX")
KINDS1 = ("COPY", "NEG")


def split_fuzz(seed: int):
    """Random tasks whose inputs often name the written store through another view."""
    rng = random.Random(seed)
    k = rng.choice((1, 2, 3))
    t = rng.choice((3, 4, 5))
    two_d = rng.random() < 0.3
    pad = 2
    ev = []
    shapes = []
    for sid in range(3):
        shape = (k * t + pad, t + pad) if two_d else (k * t + pad,)
        ev.append(CreateStore(sid, shape))
        shapes.append(shape)
    ev.append(CreateStore(3, ()))
    pid = 0
    parts = {}

    def part(sid, off):
        nonlocal pid
        key = (sid, off)
        if key not in parts:
            tile = (t, t) if two_d else (t,)
            ev.append(CreatePartition(pid, sid, "tiling", tile, off, _ident(len(tile))))
            parts[key] = pid
            pid += 1
        return parts[key]

    ev.append(CreatePartition(1000, 3, "none"))
    launch = (k, 1) if two_d else (k,)

    def off():
        return (rng.randint(0, pad), rng.randint(0, pad)) if two_d else (rng.randint(0, pad),)

    for _ in range(rng.randint(4, 10)):
        w = rng.randrange(3)
        wo = off()
        r = rng.random()
        if r < 0.12:
            src = rng.randrange(3)
            ev.append(TaskEvent("DOT", launch, ((src, part(src, off()), "R"), (w, part(w, wo), "R"),
                                                (3, 1000, "Rd"))))
        elif r < 0.25:
            ev.append(TaskEvent("AXPY", launch, ((w if rng.random() < 0.6 else rng.randrange(3), part(w, off()), "R"),
                                                 (w, part(w, wo), "RW")), (("w", rng.choice((-1.0, 2.0, 0.5))),)))
        elif r < 0.45:
            src = w if rng.random() < 0.6 else rng.randrange(3)
            so = wo if rng.random() < 0.4 else off()
            ev.append(TaskEvent(rng.choice(KINDS1), launch, ((src, part(src, so), "R"), (w, part(w, wo), "W"))))
        else:
            a = w if rng.random() < 0.5 else rng.randrange(3)
            b = w if rng.random() < 0.5 else rng.randrange(3)
            ao = wo if rng.random() < 0.4 else off()
            ev.append(TaskEvent(rng.choice(KINDS2), launch, ((a, part(a, ao), "R"), (b, part(b, off()), "R"),
                                                            (w, part(w, wo), "W"))))
        if rng.random() < 0.3:
            ev.append(Flush())
    ev.append(Flush())
    return ev


def error_case(name, events, cfg_name):
    """The reference raised ArenaViolationError: keep the trace up to the failing
    ``_execute`` (the recorder appends before executing) and the error type."""
    from diffusekit.executor import ArenaViolationError
    from diffusekit.pipeline import Session, SessionConfig, run_events
    from make_golden import builtins
    from refcapture import attach_recorder

    session = Session(SessionConfig(**CONFIGS[cfg_name]), builtins=builtins())
    trace = attach_recorder(session)
    try:
        run_events(session, events)
    except ArenaViolationError:
        trace.meta["name"] = f"{name}/{cfg_name}"
        return {"name": f"{name}/{cfg_name}", "trace": trace.to_json(), "final": {}, "error": "ArenaViolationError"}
    raise AssertionError("expected ArenaViolationError")


def one(name, events, cfg):
    from diffusekit.executor import ArenaViolationError

    try:
        return case_from_events(name, events, cfg)
    except ArenaViolationError:
        return error_case(name, events, cfg)


def main():
    cases = []
    for name, events in hand_streams().items():
        for cfg in ("fused", "unfused", "isolated"):
            cases.append(one(name, events, cfg))
    n = 0
    for seed in range(120):
        ev = split_fuzz(seed)
        for cfg in ("fused", "unfused", "isolated"):
            try:
                cases.append(one(f"split{seed}", ev, cfg))
                n += 1
            except ValueError as e:  # a stream the reference itself rejects
                print(f"split{seed}/{cfg}: reference rejected: {e}")
    for c in cases:
        if c["name"].endswith("/isolated"):
            c["trace"]["meta"]["isolated"] = True
    write(os.path.join(HERE, "alias_streams.json.gz"), cases)
    print(f"{n} fuzz cases, {sum(1 for c in cases if 'error' in c)} raising ArenaViolationError")


if __name__ == "__main__":
    main()
