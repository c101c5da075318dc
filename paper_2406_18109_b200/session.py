"""Drop-in ``Session`` whose execution runs on B200 (requires ``diffusekit``).

``GpuSession`` subclasses the reference ``Session`` (pipeline.py:128-373) and
overrides only what the north star changes:

* ``_execute`` (pipeline.py:312-345): identical report bookkeeping (prefix,
  temporaries, static traffic, kernel stats), then the fused or plain task is
  lowered once per ``Kernel`` object and handed to the device executor;
* ``heap`` (pipeline.py:141): a :class:`GpuHeap` with the reference Heap API
  (executor.py:40-79) over device stores;
* ``_maybe_free`` (pipeline.py:371-373) is inherited and reaches
  ``GpuHeap.free`` -> stream-ordered release.

The front end -- windowing, fusion constraints, temporaries, memoization,
kernel composition -- is the reference's, untouched.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .errors import ArenaViolation, BackendError, BoundsError, PrivilegeError, UnknownTaskKind
from .executor import BUILTIN_KINDS, Executor
from .ir import lower_kernel, lower_task

from diffusekit import executor as _ref_exec  # noqa: E402  (the reference front end is required here)
from diffusekit import kernels as _ref_kernels  # noqa: E402
from diffusekit.pipeline import Session as _RefSession  # noqa: E402


class _Arrays:
    """``Heap.arrays`` look-alike: item assignment uploads (test_executor.py:89-91)."""

    def __init__(self, heap: "GpuHeap") -> None:
        self._heap = heap

    def __setitem__(self, sid: int, value) -> None:
        a = np.asarray(value, dtype=np.float64)
        sess = self._heap.session
        if sess is not None and sess._is_pinned(a):
            # a pinned host array: the store's contents are defined now, the copy is
            # made by the first window that reads it (streamed with its kernel)
            sess._host_in[sid] = a
            sess._out_fresh.discard(sid)
            return
        if sess is not None:
            sess._host_in.pop(sid, None)
            sess._out_fresh.discard(sid)
        self._heap.ex.upload(sid, a)

    def __getitem__(self, sid: int) -> np.ndarray:
        if not self._heap.materialized(sid):
            raise KeyError(sid)
        return self._heap.get(sid)

    def __contains__(self, sid: int) -> bool:
        return self._heap.materialized(sid)

    def pop(self, sid: int, default=None):
        if sid in self:
            v = self[sid]
            self._heap.free(sid)
            return v
        return default


class GpuHeap:
    """Reference ``Heap`` API over device-resident stores."""

    def __init__(self, executor: Executor, session: "GpuSession | None" = None) -> None:
        self.ex = executor
        self.session = session
        self.arrays = _Arrays(self)

    def get(self, store_id: int, out: np.ndarray | None = None) -> np.ndarray:
        """The store's contents (``Heap.get``); ``out`` (backend extension): copy into this
        full-store array instead of a new one -- pinned memory makes the copy a DMA.  A store
        a streamed window already copied back into ``out`` (``GpuSession.stream_out``) is
        not copied again."""
        sess = self.session
        if sess is not None:
            host = sess._host_in.get(store_id)
            if host is not None:
                if out is None:
                    return np.array(host, copy=True)
                out[...] = host
                return out
            if store_id in sess._out_fresh:
                self.ex.sync()
                host = sess._host_out[store_id]
                if out is None:
                    return np.array(host, copy=True)
                if out is not host:
                    out[...] = host
                return out
        if out is not None:
            return self.ex.download(store_id, out=out)
        return self.ex.get(store_id)

    def materialized(self, store_id: int) -> bool:
        if self.session is not None and store_id in self.session._host_in:
            return True
        return self.ex.materialized(store_id)

    def free(self, store_id: int) -> None:
        if self.session is not None:
            self.session._host_in.pop(store_id, None)
            self.session._out_fresh.discard(store_id)
        self.ex.free(store_id)

    def digest(self, ids: Sequence[int]) -> dict[int, bytes]:
        return {s: self.get(s).tobytes() for s in ids}

    def dump_text(self, ids: Sequence[int]) -> str:
        lines = []
        for s in sorted(ids):
            arr = self.get(s)
            lines.append(f"store {s} shape {arr.shape}:")
            lines.append(np.array2string(arr, precision=6))
        return "\n".join(lines)


class GpuSession(_RefSession):
    """``Session`` whose ``_execute`` runs on the B200.

    ``graphs`` (default on, one GPU): launch segments that repeat -- the
    windows of a flush that all hit the launch-plan cache with identical
    bindings, as memo replays of a steady iteration do -- are relaunched as one
    CUDA graph (``Executor.drain``); ``DK_GRAPHS=0`` turns it off.

    Host-streamed windows (one GPU): a store assigned a pinned host array
    (``heap.arrays[sid] = session.pinned(...)``) is not uploaded at once; the
    first window that reads it -- if it is element-wise over rank-1 views --
    runs through :class:`streaming.HostStreamer`, its H2D copies, kernel and the
    D2H copies of stores registered with :meth:`stream_out` pipelined in chunks
    over three streams.  Any other use uploads first."""

    def __init__(self, config=None, registry=None, builtins=None, *, rank=0, world=1, device=None,
                 init=None, dtypes=None, graphs=True):
        super().__init__(config, registry, builtins)
        self.executor = Executor(
            seed=self.config.seed,
            init=init,
            dtypes=dtypes,
            rank=rank,
            world=world,
            device=device,
            shape_of=lambda sid: self.stores[sid].shape.extents,
        )
        self.heap = GpuHeap(self.executor, self)
        self._lowered: dict[int, tuple[object, object]] = {}
        self._pinned: list = []
        self._pinned_ranges: list[tuple[int, int]] = []
        self._host_in: dict[int, np.ndarray] = {}  # pinned host contents not yet copied to the device
        self._host_out: dict[int, np.ndarray] = {}  # stream_out registrations
        self._out_fresh: set[int] = set()  # stores whose _host_out copy is current
        self._streamer = None
        self.streamed_windows = 0
        self.executor.enable_graphs(graphs)

    def stream_out(self, store_id: int, host: np.ndarray) -> None:
        """Register a pinned full-store array that streamed windows writing ``store_id`` copy
        their result into (``heap.get(store_id, out=host)`` then needs no further copy)."""
        if not self._is_pinned(host):
            raise ValueError("stream_out needs an array from GpuSession.pinned()")
        self._host_out[store_id] = host

    def _is_pinned(self, a: np.ndarray) -> bool:
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
            return False
        lo = a.ctypes.data
        return any(b <= lo and lo + a.nbytes <= e for b, e in self._pinned_ranges)

    def _materialize_host(self, sids) -> None:
        for sid in sids:
            host = self._host_in.pop(sid, None)
            if host is not None:
                self.executor.upload(sid, host)

    def _try_stream(self, task, kp, temp_positions) -> bool:
        """Run the window through the host streamer if it reads pending host inputs and can be."""
        ins = {a.store for j, a in enumerate(task.args) if j not in temp_positions and a.store in self._host_in}
        if not ins:
            return False
        writes = {a.store for j, a in enumerate(task.args) if j not in temp_positions and a.writes}
        if (kp is None or self.executor.world != 1 or ins & writes or any(a.reduces for a in task.args)
                or any(len(self.stores[a.store].shape.extents) != 1
                       for j, a in enumerate(task.args) if j not in temp_positions)):
            return False
        from .errors import UnsupportedError
        from .streaming import HostStreamer

        if self._streamer is None:
            self._streamer = HostStreamer(self.executor, chunks=64)
        outs = {sid: self._host_out[sid] for sid in writes if sid in self._host_out}
        try:
            self._streamer.run(task, kp, temp_positions, {sid: self._host_in[sid] for sid in ins}, outs)
        except UnsupportedError:
            return False
        for sid in ins:
            del self._host_in[sid]
        self._out_fresh.difference_update(writes)
        self._out_fresh.update(outs)
        self.streamed_windows += 1
        return True

    def _flush(self, explicit: bool) -> None:  # pipeline.py:194-240, unchanged; then end the launch segment
        try:
            super()._flush(explicit)
        finally:
            self.executor.drain()

    def close(self) -> None:
        """Release the device stores, graphs and pinned host buffers of this session."""
        self._host_in.clear()
        self._host_out.clear()
        self._out_fresh.clear()
        self.executor.close()
        for p in self._pinned:
            self.executor.lib.dk_host_free(p)
        self._pinned.clear()

    def pinned(self, shape, dtype=np.float64) -> np.ndarray:
        """A host array in page-locked memory (fast, asynchronous copies to and from the heap)."""
        from .streaming import pinned

        a, p = pinned(self.executor, tuple(shape), dtype)
        self._pinned.append(p)
        self._pinned_ranges.append((a.ctypes.data, a.ctypes.data + a.nbytes))
        return a

    def _lower(self, kernel, fused: bool):
        hit = self._lowered.get(id(kernel))
        if hit is not None and hit[0] is kernel:
            return hit[1]
        kp = lower_kernel(kernel, fused)
        self._lowered[id(kernel)] = (kernel, kp)
        return kp

    def _execute(self, plan, fr) -> None:  # pipeline.py:312-345
        fr.fused_prefixes.append(plan.f)
        fr.temporaries.extend(sorted(plan.temp_stores))
        kernel = plan.kernel
        names_fused = kernel is not None
        if kernel is None and self.registry.has(plan.task.kind):
            kernel = self.registry.generate(plan.task)
        if kernel is not None:
            loads, stores = self._traffic(kernel, plan.task, plan.temp_positions, names_fused)
            fr.loads += loads
            fr.stores += stores
            fr.kernel_stats.append((plan.f, len(kernel.nests), len(kernel.locals)))
        if self.config.execute:
            if kernel is None and (plan.task.kind not in self.builtins or plan.task.kind not in BUILTIN_KINDS):
                raise _ref_exec.UnknownTaskKindError(
                    f"no generator or device builtin for task kind {plan.task.kind!r}"
                )
            kp = self._lower(kernel, names_fused) if kernel is not None else None
            # execute_isolated for fused prefixes (pipeline.py:325-334): claim checks and
            # arena-combined reductions on the device path
            isolated = plan.f > 1 and self.config.isolated
            try:
                task = lower_task(plan.task)
                streamed = False
                if self._host_in:
                    streamed = not isolated and self._try_stream(task, kp, plan.temp_positions)
                    if not streamed:
                        self._materialize_host({a.store for a in task.args})
                if not streamed:
                    self._out_fresh.difference_update({a.store for a in task.args if a.writes or a.reduces})
                    self.executor.execute(task, kp, plan.temp_positions, isolated=isolated)
            except UnknownTaskKind as e:
                raise _ref_exec.UnknownTaskKindError(str(e)) from e
            except ArenaViolation as e:
                raise _ref_exec.ArenaViolationError(str(e)) from e
            except PrivilegeError as e:
                raise _ref_kernels.PrivilegeViolationError(str(e)) from e
            except BoundsError as e:
                raise _ref_kernels.OutOfBoundsError(str(e)) from e
            except BackendError as e:
                # every other backend failure is the reference's ExecutionError
                # (executor.py:28-29); the backend type stays on __cause__
                raise _ref_exec.ExecutionError(f"{type(e).__name__}: {e}") from e
        fr.tasks_out += 1
