"""Plan traces: the front end's decisions, recorded once and replayable.

The reference front end is scale-free and never looks at data
(``test_acceptance.py:143-156``), so everything ``Session._execute``
(``pipeline.py:312-345``) receives for a stream -- the carved prefix length,
the fused ``IndexTask``, the optimized ``Kernel``, the demoted argument
positions -- can be recorded at any problem size in seconds with
``SessionConfig(execute=False)`` and replayed later.  ``tools/capture_plans.py``
records them from the unchanged reference; the GPU box, which has no copy of
the reference, replays them through the same executor entry point that
``GpuSession._execute`` uses.

A trace is a list of events:

* ``("exec", ExecStep)`` -- one ``_execute`` call;
* ``("free", sid)``      -- ``Heap.free`` issued by ``_maybe_free``
  (``pipeline.py:371-373``);
* ``("flush", explicit)`` -- end of a ``_flush`` (``pipeline.py:194-240``),
  used to cut iterations.
"""

from __future__ import annotations

import gzip
import json
from dataclasses import dataclass, field
from typing import Any

from .ir import KProg, TaskDesc, kprog_from_json, kprog_to_json, task_from_json, task_to_json


@dataclass(frozen=True)
class ExecStep:
    f: int
    task: TaskDesc
    kernel: KProg | None  # None: opaque builtin kind (executor.py:183-188)
    temp_positions: frozenset[int] = frozenset()
    temp_stores: frozenset[int] = frozenset()


@dataclass
class PlanTrace:
    seed: int
    shapes: dict[int, tuple[int, ...]]
    events: list[tuple[str, Any]]
    live: list[int] = field(default_factory=list)
    init: dict[int, dict] = field(default_factory=dict)  # InitHeap overrides by store id
    dtypes: dict[int, str] = field(default_factory=dict)  # backend dtype overrides ("i32")
    meta: dict = field(default_factory=dict)

    def execs(self) -> list[ExecStep]:
        return [e for k, e in self.events if k == "exec"]

    def iterations(self) -> list[list[tuple[str, Any]]]:
        """Events grouped by explicit flush (one group per trace iteration)."""
        out: list[list[tuple[str, Any]]] = [[]]
        for ev in self.events:
            out[-1].append(ev)
            if ev[0] == "flush" and ev[1]:
                out.append([])
        # a trailing flush of an empty buffer (Session.finish) carries no work;
        # fold exec-less groups into their predecessor so frees are not lost
        merged: list[list[tuple[str, Any]]] = []
        for g in out:
            if merged and not any(k == "exec" for k, _ in g):
                merged[-1].extend(g)
            else:
                merged.append(g)
        return [g for g in merged if g]

    # ---- serialisation ---------------------------------------------------

    def to_json(self) -> dict:
        kernels: list[dict] = []
        kidx: dict[str, int] = {}
        events = []
        for kind, ev in self.events:
            if kind == "exec":
                k = None
                if ev.kernel is not None:
                    js = json.dumps(kprog_to_json(ev.kernel), sort_keys=True)
                    if js not in kidx:
                        kidx[js] = len(kernels)
                        kernels.append(json.loads(js))
                    k = kidx[js]
                events.append(
                    [
                        "exec",
                        {
                            "f": ev.f,
                            "task": task_to_json(ev.task),
                            "kernel": k,
                            "temp_positions": sorted(ev.temp_positions),
                            "temp_stores": sorted(ev.temp_stores),
                        },
                    ]
                )
            else:
                events.append([kind, ev])
        return {
            "format": "dk-plan-1",
            "seed": self.seed,
            "shapes": {str(s): list(v) for s, v in self.shapes.items()},
            "kernels": kernels,
            "events": events,
            "live": list(self.live),
            "init": {str(s): v for s, v in self.init.items()},
            "dtypes": {str(s): v for s, v in self.dtypes.items()},
            "meta": self.meta,
        }

    @classmethod
    def from_json(cls, o: dict) -> "PlanTrace":
        if o.get("format") != "dk-plan-1":
            raise ValueError("not a dk-plan-1 trace")
        kernels = [kprog_from_json(k) for k in o["kernels"]]
        events: list[tuple[str, Any]] = []
        for kind, ev in o["events"]:
            if kind == "exec":
                events.append(
                    (
                        "exec",
                        ExecStep(
                            int(ev["f"]),
                            task_from_json(ev["task"]),
                            kernels[ev["kernel"]] if ev["kernel"] is not None else None,
                            frozenset(ev["temp_positions"]),
                            frozenset(ev["temp_stores"]),
                        ),
                    )
                )
            elif kind == "free":
                events.append(("free", int(ev)))
            else:
                events.append((kind, ev))
        return cls(
            int(o["seed"]),
            {int(s): tuple(v) for s, v in o["shapes"].items()},
            events,
            [int(s) for s in o.get("live", [])],
            {int(s): v for s, v in o.get("init", {}).items()},
            {int(s): v for s, v in o.get("dtypes", {}).items()},
            o.get("meta", {}),
        )

    def save(self, path: str) -> None:
        data = json.dumps(self.to_json(), separators=(",", ":")).encode()
        if path.endswith(".gz"):
            with gzip.open(path, "wb", compresslevel=9) as f:
                f.write(data)
        else:
            with open(path, "wb") as f:
                f.write(data)

    @classmethod
    def load(cls, path: str) -> "PlanTrace":
        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rb") as f:
            return cls.from_json(json.loads(f.read()))
