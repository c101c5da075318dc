"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This module is the checker for the B200 backend, never part of it.  Only
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product path
(``paper_2406_18109_b200``) must not import, call or fall back to anything
here.

It is a numpy restatement of the reference's execution path for one fused
(or unfused) task, operating on the backend's lowered forms
(``paper_2406_18109_b200.ir.TaskDesc`` / ``KProg``):

* ``OracleHeap``      -- ``Heap`` (diffusekit ``executor.py:40-79``);
* ``interpret``       -- ``interpret`` (``kernels.py:717-784``) with its
  whole-array path (``_eval_vec``, ``kernels.py:659-679``) and per-element
  path (``_eval_at``, ``kernels.py:682-704``);
* ``execute_step``    -- ``execute_task`` (``executor.py:163-195``) with
  ``_point_bindings`` (``executor.py:133-149``);
* builtins            -- ``_builtin_matvec``/``_builtin_norm``/``_builtin_opaque``
  (``executor.py:93-113``) plus the backend's new ``SPMV_CSR`` kind (no
  reference implementation): per row, ``acc = 0.0`` then
  ``acc = acc + vals[j] * x[cols[j]]`` left to right over the row's entries.

Parity pinning: ``tests/golden/make_golden.py`` runs the unchanged reference
on benchmark traces and a fuzz corpus and stores its final heap digests;
``tests/test_oracle_golden.py`` replays the recorded plans through this
oracle and requires byte-identical heaps.

Full-size runs (``replay(..., workers=N)``, BASELINE sizes: 32768^2 grids,
67M-row CG) split zero-offset nests into row chunks evaluated on N threads
(numpy releases the GIL) and run ``SPMV_CSR`` through the C restatement in
``oracle/csrc/spmv_csr.c``.  Every stored value is computed by exactly the same
element-wise operations as the whole-array path (a nest is only chunked when
no written view aliases another view and every bound array has the nest's
shape); only reductions change: each chunk is summed with ``np.sum`` and the
chunk sums are added in order, a different summation order from one
``np.sum`` (the device's order differs as well, so reductions are compared
at rtol).  ``tests/test_oracle_golden.py`` pins the chunked mode too.
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Mapping, Sequence

import numpy as np

from paper_2406_18109_b200.initheap import host_contents
from paper_2406_18109_b200.ir import KProg, TaskDesc, rect_of
from paper_2406_18109_b200.plan import ExecStep, PlanTrace


class OracleError(RuntimeError):
    pass


class OraclePrivilegeError(OracleError):
    pass


class OracleBoundsError(OracleError):
    pass


_UFUNC = {
    "+": np.add,
    "-": np.subtract,
    "*": np.multiply,
    "/": np.true_divide,
    "**": np.power,
    "min": np.minimum,
    "max": np.maximum,
    "lt": np.less,
    "le": np.less_equal,
    "eq": np.equal,
}


class OracleHeap:
    """Lazy store-id -> float64 array map (executor.py:40-79)."""

    def __init__(self, shapes: Mapping[int, Sequence[int]], seed: int = 0, init: Mapping[int, dict] | None = None):
        self.shapes = {int(s): tuple(v) for s, v in shapes.items()}
        self.seed = seed
        self.init = dict(init or {})
        self.arrays: dict[int, np.ndarray] = {}

    def get(self, sid: int) -> np.ndarray:
        a = self.arrays.get(sid)
        if a is None:
            a = host_contents(self.init.get(sid), self.seed, sid, self.shapes[sid])
            self.arrays[sid] = a
        return a

    def free(self, sid: int) -> None:
        self.arrays.pop(sid, None)

    def digest(self, ids: Sequence[int]) -> dict[int, bytes]:
        return {s: self.get(s).tobytes() for s in ids}


# --------------------------------------------------------------------------
# kernel interpretation
# --------------------------------------------------------------------------


def _vec(e: tuple, env: dict, scal: Sequence[float], temps: dict):
    tag = e[0]
    if tag == "ld":
        a = env[e[1]]
        return a[()] if a.ndim == 0 else a
    if tag == "sc":
        return scal[e[1]]
    if tag == "c":
        return e[1]
    if tag == "t":
        return temps[e[1]]
    if tag == "bin":
        r = _UFUNC[e[1]](_vec(e[2], env, scal, temps), _vec(e[3], env, scal, temps))
        if isinstance(r, np.ndarray) and r.dtype == bool:
            return r.astype(np.float64)
        return r
    if tag == "neg":
        return np.negative(_vec(e[1], env, scal, temps))
    return np.where(
        _vec(e[1], env, scal, temps) != 0,
        _vec(e[2], env, scal, temps),
        _vec(e[3], env, scal, temps),
    )


def _at(e: tuple, idx: tuple, env: dict, scal: Sequence[float], temps: dict):
    tag = e[0]
    if tag == "ld":
        a = env[e[1]]
        if a.ndim == 0:
            return a[()]
        pos = tuple(i + o for i, o in zip(idx, e[2]))
        if any(q < 0 or q >= n for q, n in zip(pos, a.shape)):
            raise OracleBoundsError(f"load at {pos} outside slot {e[1]} of shape {a.shape}")
        return a[pos]
    if tag == "sc":
        return np.float64(scal[e[1]])
    if tag == "c":
        return np.float64(e[1])
    if tag == "t":
        return temps[e[1]]
    if tag == "bin":
        return _UFUNC[e[1]](_at(e[2], idx, env, scal, temps), _at(e[3], idx, env, scal, temps))
    if tag == "neg":
        return np.negative(_at(e[1], idx, env, scal, temps))
    c = _at(e[1], idx, env, scal, temps)
    return _at(e[2] if c != 0 else e[3], idx, env, scal, temps)


def _loads(e: tuple):
    tag = e[0]
    if tag == "ld":
        yield e
    elif tag == "bin":
        yield from _loads(e[2])
        yield from _loads(e[3])
    elif tag == "neg":
        yield from _loads(e[1])
    elif tag == "sel":
        for x in e[1:]:
            yield from _loads(x)


def _zero_offsets(stmts) -> bool:
    for st in stmts:
        if st[0] == "store" and any(st[2]):
            return False
        e = st[3] if st[0] == "store" else st[2]
        if any(ld[2] and any(ld[2]) for ld in _loads(e)):
            return False
    return True


def interpret(
    kp: KProg,
    bufs: Mapping[int, np.ndarray],
    scalars: Sequence[float],
    local_shapes: Mapping[int, Sequence[int]],
) -> dict[int, np.ndarray]:
    """Run ``kp`` in place over slot-indexed arrays; returns the locals."""
    env: dict[int, np.ndarray] = dict(bufs)
    for i, s in enumerate(kp.slots):
        if s.local:
            if i not in local_shapes:
                raise OracleError(f"no shape for local buffer {s.name}")
            env[i] = np.zeros(tuple(local_shapes[i]), dtype=np.float64)
        elif i not in env:
            raise OracleError(f"missing binding for {s.name}")

    def writable(slot: int) -> bool:
        p = kp.slots[slot].priv
        return p is None or p in ("W", "RW")

    def reducible(slot: int) -> bool:
        p = kp.slots[slot].priv
        return p is None or p in ("W", "RW", "Rd")

    with np.errstate(all="ignore"):
        for dom, _rank, stmts in kp.nests:
            bounds = env[dom].shape
            if _zero_offsets(stmts):
                temps: dict[int, object] = {}
                for st in stmts:
                    if st[0] == "set":
                        temps[st[1]] = _vec(st[2], env, scalars, temps)
                    elif st[0] == "store":
                        if not writable(st[1]):
                            raise OraclePrivilegeError(f"store to read-only {kp.slots[st[1]].name}")
                        v = _vec(st[3], env, scalars, temps)
                        env[st[1]][...] = np.broadcast_to(v, bounds) if np.ndim(v) == 0 else v
                    else:
                        if not reducible(st[1]):
                            raise OraclePrivilegeError(f"reduce into read-only {kp.slots[st[1]].name}")
                        v = _vec(st[2], env, scalars, temps)
                        env[st[1]][()] += np.sum(v) if np.ndim(v) else v * np.prod(bounds)
            else:
                for idx in np.ndindex(*bounds):
                    temps = {}
                    for st in stmts:
                        if st[0] == "set":
                            temps[st[1]] = _at(st[2], idx, env, scalars, temps)
                        elif st[0] == "store":
                            if not writable(st[1]):
                                raise OraclePrivilegeError(f"store to read-only {kp.slots[st[1]].name}")
                            a = env[st[1]]
                            pos = tuple(i + o for i, o in zip(idx, st[2]))
                            if any(q < 0 or q >= n for q, n in zip(pos, a.shape)):
                                raise OracleBoundsError(f"store at {pos} outside {a.shape}")
                            a[pos] = _at(st[3], idx, env, scalars, temps)
                        else:
                            if not reducible(st[1]):
                                raise OraclePrivilegeError(f"reduce into read-only {kp.slots[st[1]].name}")
                            env[st[1]][()] += _at(st[2], idx, env, scalars, temps)
    return {i: env[i] for i, s in enumerate(kp.slots) if s.local}


# --------------------------------------------------------------------------
# builtins (opaque kinds)
# --------------------------------------------------------------------------

Builtin = Callable[[TaskDesc, list], None]


def _matvec(task: TaskDesc, bufs: list) -> None:
    bufs[2][...] = bufs[0] @ bufs[1]


def _norm(task: TaskDesc, bufs: list) -> None:
    bufs[1][()] += float(np.sum(bufs[0] * bufs[0]))


def _opaque(task: TaskDesc, bufs: list) -> None:
    for i, a in enumerate(task.args):
        if a.writes:
            bufs[i][...] += 1.0


def spmv_csr_rows(rowptr: np.ndarray, cols: np.ndarray, vals: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Left-to-right per-row CSR product, vectorised across rows."""
    rp = rowptr.reshape(-1).astype(np.int64)
    cl = cols.reshape(-1).astype(np.int64)
    vl = vals.reshape(-1)
    xf = x.reshape(-1)
    nrows = rp.size - 1
    start, count = rp[:-1], rp[1:] - rp[:-1]
    acc = np.zeros(nrows, dtype=np.float64)
    for k in range(int(count.max()) if nrows else 0):
        live = count > k
        j = start[live] + k
        acc[live] = acc[live] + vl[j] * xf[cl[j]]
    return acc


_CLIB = None


def _clib():
    """oracle/liboracle.so (built by oracle/build.py), or None."""
    global _CLIB
    if _CLIB is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
        if not os.path.exists(path):
            _CLIB = False
        else:
            lib = ctypes.CDLL(path)
            f = lib.oracle_spmv_csr_f64idx
            f.restype = None
            f.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int]
            _CLIB = lib
    return _CLIB or None


def spmv_csr_rows_c(rowptr, cols, vals, x, nthreads: int) -> np.ndarray:
    """spmv_csr_rows through the C restatement (same per-row order and roundings)."""
    lib = _clib()
    if lib is None:
        raise OracleError("oracle/liboracle.so is not built (python oracle/build.py)")
    arrs = [np.ascontiguousarray(a.reshape(-1), dtype=np.float64) for a in (rowptr, cols, vals, x)]
    nrows = arrs[0].size - 1
    y = np.empty(max(nrows, 0), dtype=np.float64)
    if nrows > 0:
        lib.oracle_spmv_csr_f64idx(*(a.ctypes.data for a in arrs), y.ctypes.data, nrows, int(nthreads))
    return y


def _spmv_csr(task: TaskDesc, bufs: list) -> None:
    # args: rowptr (1, t+1) R, cols (1, nnz) R, vals (1, nnz) R, x (NonePart) R, y (t,) W
    if _WORKERS > 1 and bufs[4].size >= (1 << 16) and _clib() is not None:
        y = spmv_csr_rows_c(bufs[0], bufs[1], bufs[2], bufs[3], _WORKERS)
    else:
        y = spmv_csr_rows(bufs[0], bufs[1], bufs[2], bufs[3])
    bufs[4][...] = y.reshape(bufs[4].shape)


def default_builtins() -> dict[str, Builtin]:
    return {"MATVEC": _matvec, "SPMV": _matvec, "NORM": _norm, "OPAQUE": _opaque, "SPMV_CSR": _spmv_csr}


# --------------------------------------------------------------------------
# task execution and replay
# --------------------------------------------------------------------------


def _view(a: np.ndarray, rect) -> np.ndarray:
    lo, hi = rect
    if not lo:
        return a
    return a[tuple(slice(l, h) for l, h in zip(lo, hi))]


_WORKERS = 1
_CHUNK_ELEMS = 1 << 22


def _same_view(a: np.ndarray, b: np.ndarray) -> bool:
    ia, ib = a.__array_interface__, b.__array_interface__
    return ia["data"][0] == ib["data"][0] and a.shape == b.shape and a.strides == b.strides


def _nest_chunkable(kp: KProg, nest, bufs: Mapping[int, np.ndarray]) -> bool:
    dom, _rank, stmts = nest
    if not _zero_offsets(stmts) or dom not in bufs:
        return False
    shape = bufs[dom].shape
    if len(shape) == 0 or shape[0] < 2:
        return False
    used, stored, reduced, loaded0 = set(), set(), set(), set()
    for st in stmts:
        e = st[3] if st[0] == "store" else st[2]
        for ld in _loads(e):
            used.add(ld[1])
            if bufs.get(ld[1]) is not None and bufs[ld[1]].ndim == 0:
                loaded0.add(ld[1])
        if st[0] == "store":
            stored.add(st[1])
            used.add(st[1])
        elif st[0] == "reduce":
            reduced.add(st[1])
    for i in used:
        if i not in bufs:
            return False  # a task-local buffer
        if bufs[i].ndim and bufs[i].shape != shape:
            return False  # broadcasting between ranks: keep the whole-array path
    for i in reduced:
        if i not in bufs or bufs[i].ndim != 0 or i in loaded0 or i in stored:
            return False
        if any(np.may_share_memory(bufs[i], bufs[j]) for j in used):
            return False
    for w in stored:
        for j in used:
            if j != w and np.may_share_memory(bufs[w], bufs[j]) and not _same_view(bufs[w], bufs[j]):
                return False
    return True


def _interpret_chunked(kp: KProg, bufs: dict, scalars, pool: ThreadPoolExecutor) -> None:
    """``interpret`` for kernels without locals, nest by nest, row chunks on ``pool``."""
    for nest in kp.nests:
        dom, rank, stmts = nest
        if not _nest_chunkable(kp, nest, bufs):
            one = KProg(kp.slots, kp.scalar_names, kp.ntemps, (nest,), kp.fused_names)
            interpret(one, bufs, scalars, {})
            continue
        n0 = bufs[dom].shape[0]
        inner = int(np.prod(bufs[dom].shape[1:])) if bufs[dom].ndim > 1 else 1
        rows = max(1, min(_CHUNK_ELEMS // max(inner, 1), -(-n0 // (4 * _WORKERS))))
        bounds = [(r, min(n0, r + rows)) for r in range(0, n0, rows)]
        red = [k for k, st in enumerate(stmts) if st[0] == "reduce"]
        # each reduce statement gets a private 0-d arena per chunk
        slots = list(kp.slots)
        new_stmts = []
        arena_of = {}
        for k, st in enumerate(stmts):
            if st[0] == "reduce":
                arena_of[k] = len(slots)
                from paper_2406_18109_b200.ir import Slot

                slots.append(Slot(f"rd{k}", -1, False, "Rd", 0))
                new_stmts.append(("reduce", arena_of[k], st[2]))
            else:
                new_stmts.append(st)
        kc = KProg(tuple(slots), kp.scalar_names, kp.ntemps, ((dom, rank, tuple(new_stmts)),), kp.fused_names)

        def run(b, kc=kc):
            r0, r1 = b
            sub = {i: (a[r0:r1] if a.ndim else a) for i, a in bufs.items()}
            arenas = {arena_of[k]: np.zeros(()) for k in red}
            sub.update(arenas)
            interpret(kc, sub, scalars, {})
            return [float(arenas[arena_of[k]][()]) for k in red]

        parts = list(pool.map(run, bounds))
        for idx, k in enumerate(red):
            total = 0.0
            for p in parts:
                total = total + p[idx]
            bufs[stmts[k][1]][()] += total


def execute_step(step: ExecStep, heap: OracleHeap, builtins: Mapping[str, Builtin] | None = None) -> None:
    task = step.task
    shapes = heap.shapes
    if step.kernel is None:
        builtins = builtins or default_builtins()
        fn = builtins.get(task.kind)
        if fn is None:
            raise OracleError(f"no builtin for task kind {task.kind!r}")
        for p in task.points():
            bufs = [_view(heap.get(a.store), rect_of(shapes[a.store], a.part, p)) for a in task.args]
            fn(task, bufs)
        return
    kp = step.kernel
    if len(kp.scalar_names) != len(task.scalars):
        raise OracleError("scalar arity mismatch")
    for p in task.points():
        bufs: dict[int, np.ndarray] = {}
        lshapes: dict[int, tuple] = {}
        for i, s in enumerate(kp.slots):
            a = task.args[s.arg]
            r = rect_of(shapes[a.store], a.part, p)
            if s.local:
                lshapes[i] = tuple(max(0, h - l) for l, h in zip(*r))
            else:
                bufs[i] = _view(heap.get(a.store), r)
        if _POOL is not None and not lshapes:
            _interpret_chunked(kp, bufs, task.scalars, _POOL)
        else:
            interpret(kp, bufs, task.scalars, lshapes)


_POOL: ThreadPoolExecutor | None = None


class parallel:
    """``with parallel(n):`` -- chunked, threaded evaluation (full-size parity runs)."""

    def __init__(self, workers: int | None = None) -> None:
        self.workers = workers or os.cpu_count() or 1

    def __enter__(self):
        global _POOL, _WORKERS
        self._saved = (_POOL, _WORKERS)
        if self.workers > 1:
            _WORKERS = self.workers
            _POOL = ThreadPoolExecutor(self.workers)
        return self

    def __exit__(self, *exc):
        global _POOL, _WORKERS
        if _POOL is not None and _POOL is not self._saved[0]:
            _POOL.shutdown()
        _POOL, _WORKERS = self._saved
        return False


def replay(trace: PlanTrace, events=None, heap: OracleHeap | None = None, builtins=None,
           workers: int = 1) -> OracleHeap:
    heap = heap or OracleHeap(trace.shapes, trace.seed, trace.init)
    with parallel(workers):
        for kind, ev in (events if events is not None else trace.events):
            if kind == "exec":
                execute_step(ev, heap, builtins)
            elif kind == "free":
                heap.free(ev)
    return heap
