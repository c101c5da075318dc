"""Record what the unchanged reference front end hands ``Session._execute``.

Runs only in the build container (it imports ``diffusekit`` from the
read-only reference tree or from ``baseline/_ref``).  Wraps one ``Session``
instance -- no reference file is modified -- so that every
``_execute(plan, fr)`` (``pipeline.py:312-345``), every ``Heap.free``
reached through ``_maybe_free`` (``pipeline.py:371-373``) and every
``_flush`` (``pipeline.py:194-240``) is appended to a
:class:`paper_2406_18109_b200.plan.PlanTrace`.
"""

from __future__ import annotations

import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)


def import_reference():
    """Import ``diffusekit`` without writing into the reference tree."""
    sys.dont_write_bytecode = True
    for cand in ("/root/reference/pkg/src", os.path.join(_REPO, "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "diffusekit")) and cand not in sys.path:
            sys.path.insert(0, cand)
            break
    import diffusekit  # noqa: F401

    return diffusekit


from paper_2406_18109_b200.ir import lower_kernel, lower_task  # noqa: E402
from paper_2406_18109_b200.plan import ExecStep, PlanTrace  # noqa: E402


def attach_recorder(session) -> PlanTrace:
    """Start recording ``session``'s executor calls into a new PlanTrace."""
    trace = PlanTrace(seed=session.config.seed, shapes={}, events=[])
    orig_execute = session._execute
    orig_flush = session._flush
    orig_free = session.heap.free
    kcache: dict[int, object] = {}

    def note_shapes(task) -> None:
        for a in task.args:
            trace.shapes.setdefault(a.store, tuple(session.stores[a.store].shape.extents))

    def rec_execute(plan, fr):
        task = plan.task
        note_shapes(task)
        fused = plan.kernel is not None
        kernel = plan.kernel
        if kernel is None and session.registry.has(task.kind):
            kernel = session.registry.generate(task)
        kp = None
        if kernel is not None:
            key = id(kernel) if fused else None
            if key is not None and key in kcache:
                kp = kcache[key]
            else:
                from diffusekit.kernels import kernel_text

                kp = lower_kernel(kernel, fused)
                object.__setattr__(kp, "text", kernel_text(kernel))
                if key is not None:
                    kcache[key] = kp
        trace.events.append(
            (
                "exec",
                ExecStep(
                    plan.f,
                    lower_task(task),
                    kp,
                    frozenset(plan.temp_positions),
                    frozenset(plan.temp_stores),
                ),
            )
        )
        return orig_execute(plan, fr)

    def rec_flush(explicit):
        r = orig_flush(explicit)
        trace.events.append(("flush", bool(explicit)))
        return r

    def rec_free(sid):
        trace.events.append(("free", int(sid)))
        return orig_free(sid)

    session._execute = rec_execute
    session._flush = rec_flush
    session.heap.free = rec_free
    # shapes of every store, including ones only ever dropped
    orig_create = session.create_store

    def rec_create(store_id, extents):
        st = orig_create(store_id, extents)
        trace.shapes[int(store_id)] = tuple(int(e) for e in extents)
        return st

    session.create_store = rec_create
    return trace


def record_events(events, config, builtins=None, init=None, heap_setup=None):
    """Run a reference Session over ``events`` while recording; returns (session, report, trace)."""
    dk = import_reference()
    from diffusekit.pipeline import Session, run_events

    session = Session(config, builtins=builtins)
    trace = attach_recorder(session)
    if init:
        from paper_2406_18109_b200.initheap import host_contents

        orig_get = session.heap.get

        def init_get(sid):
            if sid not in session.heap.arrays and sid in init:
                shape = session.stores[sid].shape.extents
                session.heap.arrays[sid] = host_contents(init[sid], config.seed, sid, shape)
            return orig_get(sid)

        session.heap.get = init_get
    if heap_setup is not None:
        heap_setup(session)
    report = run_events(session, events)
    trace.live = session.live_store_ids()
    trace.init = dict(init or {})
    trace.meta["report"] = {
        "tasks_in": report.tasks_in,
        "tasks_out": report.tasks_out,
        "fused_prefixes": list(report.fused_prefixes),
        "temporaries_eliminated": list(report.temporaries_eliminated),
        "loads": report.loads,
        "stores": report.stores,
        "kernel_stats": [list(ks) for fr in report.per_flush for ks in fr.kernel_stats],
    }
    return session, report, trace
