"""Host-streamed execution of an elementwise fused window (copy / compute overlap).

When a window's inputs start in host memory and its outputs are wanted back on
the host (the ``e2e`` path: a batch of options priced per call), the launch is
cut into chunks along its element range and pipelined over three streams:

    s_in : H2D of chunk c's inputs          -> event in[c]
    s_k  : waits in[c], fused kernel on c   -> event k[c]
    s_out: waits k[c], D2H of chunk c's out -> event out[c]

so PCIe H2D, kernels and D2H overlap (PCIe is full duplex) instead of running
back to back.  Elementwise means: every nest is rank-1, no reductions and no
offset loads -- exactly the windows whose per-element semantics make any
chunking legal (kernels.py:749-765).  Host arrays must be pinned
(``dk_host_alloc``) for the copies to be asynchronous.
"""

from __future__ import annotations

from ctypes import byref, c_uint64

import numpy as np

from .errors import UnsupportedError
import os

from .ir import KProg, TaskDesc, rect_of
from .runtime import check, dk_view


class HostStreamer:
    def __init__(self, ex, chunks: int = 8) -> None:
        self.ex = ex
        self.chunks = max(1, int(os.environ.get("DK_STREAM_CHUNKS", chunks)))
        lib = ex.lib
        self.main = ex.stream()
        self.streams = []
        for _ in range(3):
            s = c_uint64()
            check(lib.dk_stream_new(byref(s)))
            self.streams.append(s.value)
        self._events: list[int] = []
        self._last_k = None
        self._last_out = None
        self._main_ev = None

    def _event(self, i: int) -> int:
        while len(self._events) <= i:
            e = c_uint64()
            check(self.ex.lib.dk_event_new(byref(e)))
            self._events.append(e.value)
        return self._events[i]

    @staticmethod
    def _check(kp: KProg) -> None:
        for dom, rank, stmts in kp.nests:
            for st in stmts:
                if st[0] == "reduce":
                    raise UnsupportedError("host streaming needs an elementwise window (no reductions)")
                if st[0] == "store" and any(st[2]):
                    raise UnsupportedError("host streaming needs zero offsets")

    def run(self, task: TaskDesc, kp: KProg, temp_positions, inputs: dict, outputs: dict) -> None:
        """Execute one window; ``inputs``/``outputs`` map store ids to full-store host arrays."""
        ex, lib = self.ex, self.ex.lib
        self._check(kp)
        h, _ = ex.kernel_handle(kp)
        scal = ex._scalars(task.scalars)
        s_in, s_k, s_out = self.streams
        pts = list(task.points())
        mine = [i for i in range(len(pts)) if ex.point_rank(i, len(pts)) == ex.rank]
        n_ev = 0
        # everything already enqueued on the executor's main stream (earlier windows
        # reading these stores, uploads, frees) happens before this window's H2D
        # and kernels
        if self._main_ev is None:
            e = c_uint64()
            check(lib.dk_event_new(byref(e)))
            self._main_ev = e.value
        check(lib.dk_set_stream(self.main))
        check(lib.dk_event_record(self._main_ev))
        check(lib.dk_set_stream(s_in))
        check(lib.dk_stream_wait_event(self._main_ev))
        check(lib.dk_set_stream(s_k))
        check(lib.dk_stream_wait_event(self._main_ev))
        check(lib.dk_set_stream(self.main))
        # WAR across calls: inputs may be overwritten only after the previous kernels,
        # outputs only after the previous D2H
        if self._last_k is not None:
            check(lib.dk_set_stream(s_in))
            check(lib.dk_stream_wait_event(self._last_k))
            check(lib.dk_set_stream(s_k))
            check(lib.dk_stream_wait_event(self._last_out))
        try:
            for i in mine:
                p = pts[i]
                rects = [rect_of(ex.shape(task.args[s.arg].store), task.args[s.arg].part, p) for s in kp.slots]
                lens = {r[1][0] - r[0][0] for s, r in zip(kp.slots, rects) if len(r[0]) == 1}
                if len(lens) != 1 or any(len(r[0]) > 1 for r in rects):
                    raise UnsupportedError("host streaming needs rank-1 views of equal length")
                n = lens.pop()
                step = max(2, (n // self.chunks + 1) // 2 * 2)
                recs = [ex.rec(task.args[s.arg].store) if not s.local else None for s in kp.slots]
                for s, r, rec in zip(kp.slots, rects, recs):
                    if s.local:
                        raise UnsupportedError("host streaming does not allocate task-local buffers")
                    ex._ensure(rec, r)
                for a in range(0, n, step):
                    b = min(n, a + step)
                    ev_in, ev_k, ev_out = self._event(n_ev), self._event(n_ev + 1), self._event(n_ev + 2)
                    n_ev += 3
                    check(lib.dk_set_stream(s_in))
                    for sid, host in inputs.items():
                        for s, r, rec in zip(kp.slots, rects, recs):
                            if rec.sid == sid and len(r[0]) == 1:
                                off = (r[0][0] + a) * rec.esize
                                check(lib.dk_memcpy_h2d(rec.base + off, host.ctypes.data + off, (b - a) * rec.esize))
                                break
                    check(lib.dk_event_record(ev_in))
                    check(lib.dk_set_stream(s_k))
                    check(lib.dk_stream_wait_event(ev_in))
                    views = (dk_view * len(kp.slots))()
                    for si, (r, rec) in enumerate(zip(rects, recs)):
                        v = ex.view(rec, r)
                        if len(r[0]) == 1:
                            v.ptr += a * rec.esize
                            v.ext[0] = b - a
                        views[si] = v
                    check(lib.dk_launch(h, views, len(kp.slots), scal, len(task.scalars), 0))
                    check(lib.dk_event_record(ev_k))
                    check(lib.dk_set_stream(s_out))
                    check(lib.dk_stream_wait_event(ev_k))
                    for sid, host in outputs.items():
                        for s, r, rec in zip(kp.slots, rects, recs):
                            if rec.sid == sid and len(r[0]) == 1:
                                off = (r[0][0] + a) * rec.esize
                                check(lib.dk_memcpy_d2h_async(host.ctypes.data + off, rec.base + off, (b - a) * rec.esize))
                                break
                    check(lib.dk_event_record(ev_out))
                    self._last_k, self._last_out = ev_k, ev_out
        finally:
            check(lib.dk_set_stream(self.main))
        if self._last_out is not None:
            check(lib.dk_stream_wait_event(self._last_out))
            check(lib.dk_stream_wait_event(self._last_k))
        # coherence (replicated bookkeeping): every point's rank now holds the
        # inputs it uploaded and the stores its kernel wrote
        _, stored, _ = ex._access(kp)
        written = {kp.slots[i].arg for i in stored}
        for i in range(len(pts)):
            q = ex.point_rank(i, len(pts))
            for j, arg in enumerate(task.args):
                if j in written or arg.store in inputs:
                    ex._wrote(arg.store, rect_of(ex.shape(arg.store), arg.part, pts[i]), q)


def pinned(ex, shape, dtype=np.float64):
    """A numpy array over pinned host memory (freed with the executor's process)."""
    import ctypes

    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = ctypes.c_void_p()
    check(ex.lib.dk_host_alloc(n, byref(p)))
    buf = (ctypes.c_char * n).from_address(p.value)
    return np.frombuffer(buf, dtype=dtype).reshape(shape), p
