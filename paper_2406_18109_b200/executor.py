"""Task executor of the B200 backend (replaces diffusekit executor.py:163-195).

One process drives one GPU.  With ``world`` processes the launch points of an
index task are mapped to ranks by their lexicographic ordinal (block
distribution; one point per GPU when the launch volume equals the world size,
PAPER.md:1496-1498).  Every rank runs the same front end and therefore sees
the same stream of launches (replicated control); each rank only executes its
own points, on stores backed in HBM only where its points touch them.

Coherence.  Per store the executor keeps, identically on every rank, the rects
each rank holds valid and the rects ever written.  Before a launch it computes
what each rank's points read (R/RW views, Rd targets, builtin inputs); missing
rects are fetched from a rank that holds them (grouped NCCL send/recv, same
plan on every rank so sends and receives pair up) or materialised from the
store's initial contents if nobody ever wrote them (the Heap's lazy
initialisation, executor.py:54-61).  Writes invalidate other ranks' copies.
Fused windows need no data from other points by construction
(fusion.py:72-122), so exchanges only happen between launches: stencil halo
rows, replicated (NonePart) reads of tile-written vectors, partial sums.

Reductions.  With one rank every reduce statement accumulates directly into
its target in point order.  With several, each point's per-statement totals are
all-gathered and every rank folds ``acc = acc + total_p`` in lexicographic
point order -- the reference's combine order (executor.py:193-195), so the
replicated target is bit-identical on all ranks.  When every rank could map
every peer's reduction board (``dk_p2p_init``), the gather is not a separate
collective: the reducing kernel's last CTA writes its point's totals into all
ranks' boards over NVLink and raises a flag there (``dk_launch_pub``); the
fold waits on the flags of its board slot (``dk_p2p_wait``).  Otherwise, and
for builtins, the totals go through an NCCL all-gather.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import byref, c_double, c_int, c_int32, c_int64, c_uint8, c_uint64
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

from . import aliasing
from . import regions as rg
from . import runtime
from .errors import ArenaViolation, BackendError, UnknownTaskKind, UnsupportedError
from .initheap import host_contents, poisson_tile, poisson_tile_layout, row_chunks
from .ir import KProg, TaskDesc, rect_of, slot_access
from .runtime import DK_F64, DK_I32, check, dk_view, i64s

BUILTIN_KINDS = ("MATVEC", "SPMV", "NORM", "OPAQUE", "SPMV_CSR")
DEVICE_INIT_MIN = 1 << 16  # stores at least this large get their initial contents from dk_pcg64_fill


@dataclass
class StoreRec:
    sid: int
    shape: tuple[int, ...]
    dtype: str  # "f64" | "i32"
    valid: list[list] = field(default_factory=list)  # per rank: disjoint rects
    written: list = field(default_factory=list)
    on_device: bool = False
    base: int = 0
    strides: tuple[int, ...] = ()
    pcg: tuple | None = None  # (elements covered, rejection breakpoints) of the default init stream

    @property
    def esize(self) -> int:
        return 8 if self.dtype == "f64" else 4

    @property
    def full(self):
        return (tuple(0 for _ in self.shape), tuple(self.shape))


@dataclass
class LaunchStats:
    launches: int = 0
    points: int = 0
    bytes_moved: int = 0
    transfers: int = 0
    inits: int = 0
    p2p_folds: int = 0  # reductions gathered through the peer-memory boards
    p2p_halos: int = 0  # transfer sets moved through the peer mailboxes
    mplan_hits: int = 0  # multi-GPU launches replayed from the plan cache


class Executor:
    """Device-side heap + launch engine for one rank."""

    def __init__(
        self,
        shapes: Mapping[int, Sequence[int]] | None = None,
        seed: int = 0,
        init: Mapping[int, dict] | None = None,
        dtypes: Mapping[int, str] | None = None,
        rank: int = 0,
        world: int = 1,
        device: int | None = None,
        shape_of=None,
        lib=None,
        fuse_spmv_dot: bool | None = None,
    ) -> None:
        # ``lib``: an object with the C-ABI's functions; only the test-suite's CPU
        # stand-in passes one.  The product always loads libdk_b200.so.
        self.lib = lib if lib is not None else runtime.load()
        self.rank = rank
        self.world = world
        self.device = rank if device is None else device
        check(self.lib.dk_init(self.device))
        self.shapes = {int(s): tuple(v) for s, v in (shapes or {}).items()}
        self.shape_of = shape_of
        self.seed = seed
        self.init = dict(init or {})
        self.dtypes = dict(dtypes or {})
        self.stores: dict[int, StoreRec] = {}
        self._kcache: dict[int, tuple[KProg, int, int]] = {}
        self._kval: dict[KProg, tuple[int, int]] = {}
        self._scal: dict[tuple, ctypes.Array] = {}
        self._acc: dict[int, tuple] = {}
        self._plans: dict[tuple, tuple] = {}  # launch-plan cache (one GPU)
        self._alias_c: dict[tuple, tuple] = {}  # (kp, args) -> does a written store have two views
        self._alias_k: dict[tuple, tuple] = {}  # rewritten kernels of identical-rect alias groups
        self._mplans: dict[tuple, dict] = {}  # launch-plan cache (several GPUs), keyed on coherence state
        self._rec: dict | None = None  # the multi-GPU plan being recorded by execute()
        self.stats = LaunchStats()
        self._comm = False
        self._p2p = False
        self._p2p_epoch = 0
        self._ts = None  # diagnostics: (device buffer, capacity, [labels]) for mark()
        self._collect = None  # fold ops being gathered for dk_p2p_wait_fold
        self._side = None  # side stream (+ events) of the overlapped SpMV halo sends
        self._side_ev = None
        # CUDA-graph relaunch of repeated launch segments (enable_graphs)
        self._graphs_on = False
        self._pending: list = []  # deferred plan-cache hits: (handle, views, scalars, nscal, nslots)
        self._seg_seen: dict[tuple, int] = {}
        self._seg_graphs: dict[tuple, int] = {}
        self.graph_stats = {"segments": 0, "graph_launches": 0, "captures": 0, "direct": 0}
        # opt-in SpMV + partial-dot epilogue (backend-only; the fusion plan is unchanged)
        if fuse_spmv_dot is None:
            fuse_spmv_dot = os.environ.get("DK_FUSE_SPMV_DOT", "0") == "1"
        self.fuse_spmv_dot = bool(fuse_spmv_dot)
        self._sd = None  # totals of the last SPMV_CSR's p.q, waiting for the window that reduces it
        self._sd_buf = (0, 0)  # (device ptr, regions): dk_spmv_csr_dot partials + ticket + total
        self.spmv_dot_stats = {"spmv": 0, "consumed": 0, "replayed": 0}  # replayed: consumers from the plan cache

    # ------------------------------------------------------------------ comm
    def init_comm(self, unique_id: bytes) -> None:
        buf = (c_uint8 * 128)(*unique_id)
        check(self.lib.dk_comm_init(self.rank, self.world, buf))
        self._comm = True
        self.enable_p2p()

    def enable_p2p(self) -> bool:
        """Collective: switch kernel reductions to the peer-memory board exchange
        if every rank mapped every peer's board (DK_P2P=0 keeps NCCL)."""
        if self.world > 1 and os.environ.get("DK_P2P", "1") != "0":
            ok = c_int(0)
            check(self.lib.dk_p2p_init(byref(ok)))
            self._p2p = bool(ok.value)
        return self._p2p

    def comm_unique_id(self) -> bytes:
        buf = (c_uint8 * 128)()
        check(self.lib.dk_comm_unique_id(buf))
        return bytes(buf)

    # ---------------------------------------------------------------- stores
    def shape(self, sid: int) -> tuple[int, ...]:
        s = self.shapes.get(sid)
        if s is None and self.shape_of is not None:
            s = tuple(self.shape_of(sid))
            self.shapes[sid] = s
        if s is None:
            raise BackendError(f"unknown store {sid}")
        return s

    def rec(self, sid: int) -> StoreRec:
        r = self.stores.get(sid)
        if r is None:
            shape = self.shape(sid)
            strides = [1] * len(shape)
            for d in range(len(shape) - 2, -1, -1):
                strides[d] = strides[d + 1] * shape[d + 1]
            r = StoreRec(sid, shape, self.dtypes.get(sid, "f64"), [[] for _ in range(self.world)], [], strides=tuple(strides))
            self.stores[sid] = r
        return r

    def _device(self, r: StoreRec) -> None:
        if r.on_device:
            return
        check(self.lib.dk_store_create(r.sid, len(r.shape), i64s(r.shape), DK_F64 if r.dtype == "f64" else DK_I32))
        p = c_uint64()
        check(self.lib.dk_store_ptr(r.sid, byref(p)))
        r.base = p.value
        r.on_device = True

    def _ensure(self, r: StoreRec, rect) -> None:
        if rg.empty(rect):
            return
        if self._rec is not None:
            self._rec["ensure"].append((r.sid, rect))
        self._device(r)
        lo, hi = rg.bbox_flat(r.shape, rect)
        check(self.lib.dk_store_ensure(r.sid, lo, hi))

    def _drop_sd(self) -> None:
        self._sd = None

    def _sd_regions(self, n: int) -> int:
        """Device buffer of ``n`` dk_spmv_csr_dot regions (SPMV_DOT_DOUBLES each, tickets zeroed
        once; the kernel leaves them zero).  Kept across launches: a pending ``_sd`` is always
        consumed or dropped before the next SpMV, and both are stream-ordered."""
        ptr, have = self._sd_buf
        if have < n:
            if ptr:
                check(self.lib.dk_scratch_free(ptr))
            have = max(4, n)
            p = c_uint64()
            check(self.lib.dk_scratch_alloc(8 * runtime.SPMV_DOT_DOUBLES * have, byref(p)))
            check(self.lib.dk_memset_zero(p.value, 8 * runtime.SPMV_DOT_DOUBLES * have))
            ptr = p.value
            self._sd_buf = (ptr, have)
        return ptr

    def free(self, sid: int) -> None:
        if self._sd is not None and sid in (self._sd["x"], self._sd["y"]):
            self._drop_sd()
        r = self.stores.pop(sid, None)
        if r is not None and r.on_device:
            self.drain()
            check(self.lib.dk_store_free(sid))

    def close(self) -> None:
        """Release every store this executor created (device state is process-global)."""
        self.drop_graphs()
        self._drop_sd()
        if self._sd_buf[0]:
            check(self.lib.dk_scratch_free(self._sd_buf[0]))
            self._sd_buf = (0, 0)
        for sid in list(self.stores):
            self.free(sid)
        check(self.lib.dk_sync())

    def materialized(self, sid: int) -> bool:
        r = self.stores.get(sid)
        return r is not None and any(r.valid[q] for q in range(self.world))

    # -------------------------------------------------- initial contents
    def _materialize_init(self, r: StoreRec, rects: list) -> None:
        """Upload the store's initial contents for ``rects`` on this rank."""
        rects = [x for x in rects if not rg.empty(x)]
        if not rects:
            return
        for x in rects:
            self._ensure(r, x)
        self.stats.inits += len(rects)
        spec = self.init.get(r.sid)
        kind = None if spec is None else spec["kind"]
        np_dtype = np.float64 if r.dtype == "f64" else np.int32
        if kind in ("zeros", "const", "poisson_invdiag") and r.dtype == "f64":
            v = {"zeros": 0.0, "poisson_invdiag": 0.25}.get(kind, float(spec.get("value", 0.0)))
            for x in rects:
                for a, b in self._flat_runs(r, x):
                    check(self.lib.dk_store_fill(r.sid, a, b, v))
            return
        if kind in ("csr_rowptr", "csr_cols", "csr_vals"):
            self._materialize_csr(r, spec, rects, np_dtype)
            return
        if (kind is None or kind == "uniform") and r.dtype == "f64" and len(r.shape) in (1, 2) \
                and int(np.prod(r.shape)) >= DEVICE_INIT_MIN and not os.environ.get("DK_HOST_INIT"):
            self._materialize_pcg(r, spec, rects)
            return
        if not r.shape:
            host = host_contents(spec, self.seed, r.sid, r.shape).astype(np_dtype)
            check(self.lib.dk_store_upload_rect(r.sid, i64s([0]), i64s([0]), host.ctypes.data))
            return
        row = 1
        for e in r.shape[1:]:
            row *= e
        row_end = max(x[1][0] for x in rects)
        for r0, r1, chunk in row_chunks(spec, self.seed, r.sid, r.shape, row_end):
            chunk = np.ascontiguousarray(chunk, dtype=np_dtype)
            base = chunk.ctypes.data - r0 * row * r.esize  # virtual full-store origin
            for x in rects:
                lo0, hi0 = max(x[0][0], r0), min(x[1][0], r1)
                if lo0 >= hi0:
                    continue
                lo = (lo0,) + x[0][1:]
                hi = (hi0,) + x[1][1:]
                check(self.lib.dk_store_upload_rect(r.sid, i64s(lo), i64s(hi), ctypes.c_void_p(base)))
            check(self.lib.dk_sync())  # the chunk buffer is reused by the generator

    def _materialize_pcg(self, r: StoreRec, spec: dict | None, rects: list) -> None:
        """Device-side PCG64: same bits as numpy's stream, only this rank's rects (csrc/dk_pcg.cu)."""
        if spec is None:
            key, kind, scale = [self.seed, r.sid], 0, 1.0
        else:
            key, kind = [int(spec.get("seed", 0)), int(spec.get("key", r.sid))], 1
            scale = float(spec["scale"]) if "scale" in spec else 1.0
        s = np.random.default_rng(key).bit_generator.state["state"]
        m64 = (1 << 64) - 1
        st = (c_uint64 * 2)(s["state"] >> 64, s["state"] & m64)
        inc = (c_uint64 * 2)(s["inc"] >> 64, s["inc"] & m64)
        breaks: list[int] = []
        if kind == 0:
            emax = max(rg.bbox_flat(r.shape, x)[1] for x in rects)
            if r.pcg is None or r.pcg[0] < emax:
                d_end = emax + 64
                while True:
                    cap = 1 << 16
                    out = (c_int64 * cap)()
                    cnt = c_int64()
                    check(self.lib.dk_pcg64_rejects(st, inc, d_end, out, cap, byref(cnt)))
                    if cnt.value > cap:
                        raise BackendError("PCG64 stream has more rejections than expected")
                    if emax + cnt.value <= d_end:
                        break
                    d_end = emax + cnt.value + 64
                qs = list(out[: cnt.value])
                r.pcg = (emax, [q - k for k, q in enumerate(qs)])
            breaks = r.pcg[1]
        barr = (c_int64 * max(len(breaks), 1))(*breaks)
        for x in rects:
            check(self.lib.dk_pcg64_fill(r.sid, i64s(x[0]), i64s(x[1]), st, inc, kind, scale, barr, len(breaks)))

    def _materialize_csr(self, r: StoreRec, spec: dict, rects: list, np_dtype) -> None:
        nx, ny, k = int(spec["nx"]), int(spec["ny"]), int(spec["k"])
        lay = poisson_tile_layout(nx, ny, k)
        which = ("csr_rowptr", "csr_cols", "csr_vals").index(spec["kind"])
        seg = lay["t"] + 1 if which == 0 else lay["nnz_max"]
        for p in range(k):
            tile_rect = ((p * seg,), ((p + 1) * seg,))
            parts = [rg.intersect(x, tile_rect) for x in rects]
            parts = [x for x in parts if not rg.empty(x)]
            if not parts:
                continue
            arr = np.ascontiguousarray(poisson_tile(nx, ny, k, p)[which], dtype=np_dtype)
            base = arr.ctypes.data - p * seg * r.esize
            for x in parts:
                check(self.lib.dk_store_upload_rect(r.sid, i64s(x[0]), i64s(x[1]), ctypes.c_void_p(base)))
            check(self.lib.dk_sync())

    def _flat_runs(self, r: StoreRec, x) -> list[tuple[int, int]]:
        """Contiguous [a, b) element runs covering rect x (row-major)."""
        shape = r.shape
        if not shape:
            return [(0, 1)]
        n = len(shape)
        inner = n - 1
        while inner > 0 and x[0][inner] == 0 and x[1][inner] == shape[inner]:
            inner -= 1
        runs = []
        outer = [range(x[0][d], x[1][d]) for d in range(inner)]
        import itertools

        for idx in itertools.product(*outer):
            a = sum(i * r.strides[d] for d, i in enumerate(idx)) + x[0][inner] * r.strides[inner]
            b = a + (x[1][inner] - x[0][inner]) * r.strides[inner]
            runs.append((a, b))
        return runs

    # ------------------------------------------------------------ coherence
    def point_rank(self, ordinal: int, volume: int) -> int:
        if self.world == 1:
            return 0
        if volume >= self.world:
            return ordinal * self.world // volume
        return ordinal

    def _satisfy(self, need: dict[int, dict[int, list]], defer: bool = False):
        """Make every rank's needed rects valid (same plan on every rank).

        ``defer``: plan (and book) the transfers but return this rank's share,
        ``[(sid, rect, src, dst)]``, for the caller to move; initialisations run now."""
        snap = {sid: [list(v) for v in self.stores[sid].valid] for sid in {s for d in need.values() for s in d}}
        transfers = []  # (sid, rect, src, dst)
        inits: dict[int, list] = {}
        for q in range(self.world):
            for sid in sorted(need.get(q, {})):
                r = self.stores[sid]
                for want in need[q][sid]:
                    missing = rg.minus([want], r.valid[q])
                    for m in missing:
                        unwritten = rg.minus([m], r.written)
                        if q == self.rank and unwritten:
                            inits.setdefault(sid, []).extend(unwritten)
                        rest = rg.minus([m], unwritten)
                        for src in range(self.world):
                            if not rest:
                                break
                            if src == q:
                                continue
                            for v in snap[sid][src]:
                                for rr in rest:
                                    piece = rg.intersect(rr, v)
                                    if not rg.empty(piece):
                                        transfers.append((sid, piece, src, q))
                                rest = rg.minus(rest, [v])
                                if not rest:
                                    break
                        if rest:
                            raise BackendError(f"coherence: store {sid} rect {rest[0]} valid nowhere")
                    r.valid[q] = rg.add(r.valid[q], want) if missing else r.valid[q]
        if inits and self._rec is not None:
            self._rec["inits"] = [(sid, list(rects)) for sid, rects in inits.items()]
        for sid, rects in inits.items():
            self._materialize_init(self.stores[sid], rects)
        mine = [t for t in transfers if self.rank in (t[2], t[3])]
        if defer:
            for sid, rect, _src, _dst in mine:
                self._ensure(self.stores[sid], rect)
                self.stats.bytes_moved += rg.volume(rect) * self.stores[sid].esize
            self.stats.transfers += len(mine)
            return mine
        if mine:
            if not self._comm:
                raise BackendError("multi-rank transfer without an initialised communicator")
            n = len(mine)
            sids = (c_int64 * n)()
            peers = (c_int32 * n)()
            dirs = (c_int32 * n)()
            los = (c_int64 * (4 * n))()
            his = (c_int64 * (4 * n))()
            for i, (sid, rect, src, dst) in enumerate(mine):
                r = self.stores[sid]
                self._ensure(r, rect)
                sids[i] = sid
                send = src == self.rank
                peers[i] = dst if send else src
                dirs[i] = 0 if send else 1
                for d in range(len(rect[0])):
                    los[4 * i + d] = rect[0][d]
                    his[4 * i + d] = rect[1][d]
                self.stats.bytes_moved += rg.volume(rect) * r.esize
            self.stats.transfers += n
            self._exchange(n, sids, peers, dirs, los, his)
            if self._rec is not None:
                nbytes = sum(rg.volume(t[1]) * self.stores[t[0]].esize for t in mine)
                self._rec["xfer"] = (n, sids, peers, dirs, los, his, nbytes)

    def _contiguous(self, sid, lo, hi) -> bool:
        """A rect of a row-major store is one contiguous span: after its first dimension with
        more than one index, every dimension is full."""
        shape = self.stores[sid].shape
        ext = [hi[d] - lo[d] for d in range(len(shape))]
        for d in range(len(shape)):
            if ext[d] > 1:
                return all(lo[e] == 0 and hi[e] == shape[e] for e in range(d + 1, len(shape)))
        return True

    def _exchange(self, n, sids, peers, dirs, los, his) -> None:
        """Move the transfer list: pairs whose rects fit a peer mailbox go through peer memory --
        by copy engine (dk_dma_send / dk_dma_recv, DK_P2P_HALO=2) or by one pack/unpack kernel
        (dk_p2p_exchange, DK_P2P_HALO=1) -- the rest through grouped NCCL send/recv.  The split is
        per peer pair and computed from the replicated plan, so both ends of a pair decide alike."""
        use = {}
        mode = os.environ.get("DK_P2P_HALO", "0")
        if self._p2p and mode in ("1", "2"):
            per = {}
            for i in range(n):
                key = (peers[i], dirs[i])
                esz = self.stores[sids[i]].esize
                vol = 1
                for d in range(len(self.stores[sids[i]].shape)):
                    vol *= max(0, his[4 * i + d] - los[4 * i + d])
                b, k = per.get(key, (0, 0))
                per[key] = (b + ((vol * esz + 15) // 16) * 16, k + 1)
            for q in {peers[i] for i in range(n)}:
                fits = all(per.get((q, d), (0, 0))[0] <= runtime.P2P_MAIL_BYTES and per.get((q, d), (0, 0))[1] <= 8
                           for d in (0, 1))
                if mode == "2":
                    fits = fits and all(self._contiguous(sids[i], los[4 * i:4 * i + 4], his[4 * i:4 * i + 4])
                                        for i in range(n) if peers[i] == q)
                use[q] = fits
        p2p_idx = [i for i in range(n) if use.get(peers[i])]
        nccl_idx = [i for i in range(n) if not use.get(peers[i])]

        def sub(idx):
            m = len(idx)
            return (m, (c_int64 * m)(*[sids[i] for i in idx]), (c_int32 * m)(*[peers[i] for i in idx]),
                    (c_int32 * m)(*[dirs[i] for i in idx]),
                    (c_int64 * (4 * m))(*[los[4 * i + d] for i in idx for d in range(4)]),
                    (c_int64 * (4 * m))(*[his[4 * i + d] for i in idx for d in range(4)]))

        if p2p_idx and mode == "2":
            # sends first: a send waits only for the ack of the message two before, never for
            # this exchange, so every rank's sends are posted before any rank waits on a receive
            for d, fn in ((0, self.lib.dk_dma_send), (1, self.lib.dk_dma_recv)):
                idx = [i for i in p2p_idx if dirs[i] == d]
                if idx:
                    m, s_, p_, _d, lo_, hi_ = sub(idx)
                    check(fn(m, s_, p_, lo_, hi_))
            self.stats.p2p_halos += 1
        elif p2p_idx:
            check(self.lib.dk_p2p_exchange(*(sub(p2p_idx) if nccl_idx else (n, sids, peers, dirs, los, his))))
            self.stats.p2p_halos += 1
        if nccl_idx:
            check(self.lib.dk_comm_exchange(*(sub(nccl_idx) if p2p_idx else (n, sids, peers, dirs, los, his))))

    def _wrote(self, sid: int, rect, q: int) -> None:
        r = self.stores[sid]
        if rg.empty(rect):
            return
        for o in range(self.world):
            if o != q and r.valid[o]:
                r.valid[o] = rg.minus(r.valid[o], [rect])
        r.valid[q] = rg.add(r.valid[q], rect)
        r.written = rg.add(r.written, rect)

    # --------------------------------------------------------------- views
    def view(self, r: StoreRec, rect) -> dk_view:
        self._device(r)  # empty views still need a base address
        v = dk_view()
        lo, hi = rect
        off = sum(l * s for l, s in zip(lo, r.strides))
        v.ptr = r.base + off * r.esize
        v.rank = len(r.shape)
        v.dtype = DK_F64 if r.dtype == "f64" else DK_I32
        for d in range(len(r.shape)):
            v.ext[d] = max(0, hi[d] - lo[d])
            v.stride[d] = r.strides[d]
        return v

    # -------------------------------------------------------------- kernels
    def kernel_handle(self, kp: KProg) -> tuple[int, int]:
        hit = self._kcache.get(id(kp))
        if hit is not None and hit[0] is kp:
            return hit[1], hit[2]
        val = self._kval.get(kp)
        if val is None:
            text = kp.wire([s.decl_rank for s in kp.slots]).encode()
            h = c_int64()
            check(self.lib.dk_kernel_compile(text, len(text), byref(h)))
            nred = sum(1 for _, _, stmts in kp.nests for st in stmts if st[0] == "reduce")
            val = (h.value, nred)
            self._kval[kp] = val
        self._kcache[id(kp)] = (kp, val[0], val[1])
        return val

    def kernel_source(self, kp: KProg) -> str:
        h, _ = self.kernel_handle(kp)
        n = c_int64()
        check(self.lib.dk_kernel_source(h, None, 0, byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(self.lib.dk_kernel_source(h, buf, n.value + 1, byref(n)))
        return buf.value.decode()

    def _scalars(self, vals: tuple[float, ...]) -> ctypes.Array:
        a = self._scal.get(vals)
        if a is None:
            a = (c_double * max(len(vals), 1))(*vals)
            if len(self._scal) > 4096:
                self._scal.clear()
            self._scal[vals] = a
        return a

    # ------------------------------------------------------------- execute
    def execute(self, task: TaskDesc, kp: KProg | None, temp_positions: Iterable[int] = (),
                isolated: bool = False) -> None:
        """Run one (fused or plain) index task: execute_task (executor.py:163-195).

        ``isolated``: execute_isolated's contract (executor.py:209-293) -- the
        per-point write-claim checks (ArenaViolation), then reductions that
        collect each point's contributions in a zeroed arena before adding it
        to the target in point order (executor.py:280-293)."""
        if kp is None and task.kind not in BUILTIN_KINDS:
            raise UnknownTaskKind(f"no generator or builtin for task kind {task.kind!r}")
        temp_positions = frozenset(temp_positions)
        use_mplan = os.environ.get("DK_MPLAN", "1") != "0"
        sd = None
        if self._sd is not None:
            sd, self._sd = self._sd, None
            if kp is None or isolated:
                sd = None
            elif self.world == 1 or not use_mplan:
                self.drain()
                self._execute_planned(task, kp, temp_positions, None, spmv_dot=sd)
                return
        if isolated:
            if kp is None:
                raise BackendError(f"isolated execution needs a kernel for kind {task.kind!r}")
            self.drain()
            self.check_isolated(task, temp_positions)
            self._execute_planned(task, kp, temp_positions, None, isolated=True)
            return
        pkey = None
        if kp is not None and self.world == 1:
            # key on the non-temporary arguments: each memo replay of a window names fresh
            # temporaries, which never reach the device
            pkey = (id(kp), task.launch, temp_positions, task.scalars,
                    tuple(a for j, a in enumerate(task.args) if j not in temp_positions))
            hit = self._plans.get(pkey)
            # valid while every store is the same record: on one GPU a store's valid
            # region only grows until it is freed, and bindings depend only on shapes
            if hit is not None and hit[0] is kp and all(self.stores.get(s) is r for s, r in hit[1]):
                h, _ = self.kernel_handle(kp)
                scal = self._scalars(task.scalars)
                for views in hit[2]:
                    if self._graphs_on:
                        self._pending.append((h, views, scal, len(task.scalars), len(kp.slots)))
                    else:
                        check(self.lib.dk_launch(h, views, len(kp.slots), scal, len(task.scalars), 0))
                self.stats.launches += 1
                self.stats.points += len(hit[2])
                return
        self.drain()
        if use_mplan:
            key, sids = self._mplan_key(task, kp, temp_positions)
            if key is not None and sd is not None:
                # a window consuming the SpMV epilogue's p.q is its own plan
                if sd["x"] not in sids or sd["y"] not in sids:
                    key = None
                else:
                    key = key + (("spmv_dot", sids.index(sd["x"]), sids.index(sd["y"]), tuple(sorted(sd["pts"]))),)
            hit = self._mplans.get(key) if key is not None else None
            if hit is not None and hit["kp"] is kp:
                self._mplan_replay(hit, task, kp, sids, sd)
                return
            self._rec = {"ok": key is not None, "xfer": None, "views": [], "fold": [], "pub": False,
                         "ensure": [], "inits": []}
            try:
                self._execute_planned(task, kp, temp_positions, pkey, spmv_dot=sd)
                if self._rec["ok"]:
                    self._mplan_store(key, sids, kp)
            finally:
                self._rec = None
            return
        self._execute_planned(task, kp, temp_positions, pkey)

    # ------------------------------------------------ diagnostics
    def trace_timestamps(self, capacity: int = 1 << 16) -> None:
        """Start recording device timestamps at mark() points (bench DK_TRACE_TS)."""
        p = c_uint64()
        check(self.lib.dk_scratch_alloc(8 * capacity, byref(p)))
        self._ts = (p.value, capacity, [])

    def mark(self, label: str) -> None:
        if self._ts is None:
            return
        buf, cap, labels = self._ts
        if len(labels) < cap:
            check(self.lib.dk_timestamp(buf, len(labels)))
            labels.append(label)

    def timestamps(self):
        """[(label, globaltimer ns)] recorded so far (synchronises)."""
        if self._ts is None:
            return []
        buf, cap, labels = self._ts
        self.sync()
        out = np.empty(max(len(labels), 1), dtype=np.uint64)
        check(self.lib.dk_memcpy_d2h(out.ctypes.data, buf, 8 * len(labels)))
        return list(zip(labels, out[: len(labels)].tolist()))

    # ------------------------------------------------ graph relaunch (f3)
    # With graphs enabled (GpuSession, one GPU), launches that hit the launch-plan
    # cache are not issued at once but collected into a segment; the segment ends
    # at the session's flush or at the first operation that is not such a hit
    # (a planned launch, a free of a device store, any host transfer or sync).
    # A segment is keyed by its exact launches (kernel handle, bound views and
    # scalars, in order).  The second time a key is seen it is captured into a
    # CUDA graph (dk_graph_*), and from then on each occurrence is one graph
    # launch.  The key is the launch parameters themselves, so a graph can only
    # ever replay launches the plan cache just decided to issue; no
    # invalidation is needed when stores are freed and recreated.
    def enable_graphs(self, on: bool = True) -> None:
        self.drain()
        self._graphs_on = bool(on) and self.world == 1 and os.environ.get("DK_GRAPHS", "1") != "0"

    def drain(self) -> None:
        """Issue the deferred launch segment (as a graph when it repeats)."""
        if not self._pending:
            return
        pend, self._pending = self._pending, []
        self.graph_stats["segments"] += 1
        key = tuple((h, bytes(v), bytes(sc)[: 8 * ns]) for h, v, sc, ns, _ in pend)
        g = self._seg_graphs.get(key)
        if g is None:
            n = self._seg_seen.get(key, 0) + 1
            if n >= 2 and len(self._seg_graphs) < 256:
                def issue():
                    for h, v, sc, ns, nsl in pend:
                        check(self.lib.dk_launch(h, v, nsl, sc, ns, 0))

                g = self.capture(issue)
                self._seg_graphs[key] = g
                self.graph_stats["captures"] += 1
                self._seg_seen.pop(key, None)
            else:
                if len(self._seg_seen) > 4096:
                    self._seg_seen.clear()
                self._seg_seen[key] = n
                for h, v, sc, ns, nsl in pend:
                    check(self.lib.dk_launch(h, v, nsl, sc, ns, 0))
                self.graph_stats["direct"] += 1
                return
        check(self.lib.dk_graph_launch(c_uint64(g)))
        self.graph_stats["graph_launches"] += 1

    def drop_graphs(self) -> None:
        self.drain()
        for g in self._seg_graphs.values():
            check(self.lib.dk_graph_destroy(c_uint64(g)))
        self._seg_graphs.clear()
        self._seg_seen.clear()

    # ------------------------------------------------ multi-GPU plan cache
    # A memo-replayed window repeats with the same launch, the same coherence
    # state of its stores (valid / written rects per rank) and -- for the
    # per-iteration scalars of CG -- fresh rank-0 stores in the same roles.
    # Stores are therefore keyed by their first-appearance index in the task's
    # arguments; the recorded transfers, initialisations, bindings (pointer =
    # store base + offset), fold and post-launch coherence state are replayed
    # onto the actual stores.  Every rank holds the same replicated state, so
    # every rank hits or misses together.
    def _mplan_key(self, task, kp, temp_positions):
        sids = []
        for j, a in enumerate(task.args):
            if j not in temp_positions and a.store not in sids:
                sids.append(a.store)
        sig = []
        for sid in sids:
            r = self.rec(sid)
            sig.append((r.shape, r.dtype, tuple(tuple(v) for v in r.valid), tuple(r.written),
                        sid if r.shape else None))  # large stores by identity, rank-0 ones by role
        cidx = {sid: c for c, sid in enumerate(sids)}
        args = tuple((cidx[a.store], a.part, a.priv) if j not in temp_positions else None
                     for j, a in enumerate(task.args))
        kid = id(kp) if kp is not None else task.kind
        return (kid, task.launch, temp_positions, task.scalars, args, tuple(sig)), sids

    def _mplan_store(self, key, sids, kp) -> None:
        rec = self._rec
        cidx = {sid: c for c, sid in enumerate(sids)}
        base = {sid: self.stores[sid].base for sid in sids if sid in self.stores}

        def canon_views(views, slots):
            out = []
            for idx, sid in slots:
                if sid not in cidx or sid not in base:
                    return None
                v = views if idx is None else views[idx]
                out.append((idx, cidx[sid], v.ptr - base[sid]))
            return (views, out)

        plan = {"kp": kp, "pub": rec["pub"], "counts": rec.get("counts")}
        vs = []
        for item in rec["views"]:
            if kp is None:
                (views, slots), n, wflags = item
                cv = canon_views(views, slots)
                vs.append(None if cv is None else (cv, n, wflags))
            else:
                vs.append(canon_views(*item))
        fold = []
        for (tv, slots), first, stride, n in rec["fold"]:
            cv = canon_views(tv, slots)
            fold.append(None if cv is None else (cv, first, stride, n))
        if any(v is None for v in vs) or any(f is None for f in fold):
            return
        if any(sid not in cidx for sid, _ in rec["ensure"]) or any(sid not in cidx for sid, _ in rec["inits"]):
            return
        ov = rec.get("overlap")
        if ov is not None:
            if any(sid not in cidx for sid, _r, _q in ov["sends"] + ov["recvs"]):
                return
            cvs = [canon_views(v, slots) for v, slots in ov["views"]]
            if any(c is None for c in cvs):
                return
            plan["overlap"] = {"sends": [(cidx[sid], r, q) for sid, r, q in ov["sends"]],
                               "recvs": [(cidx[sid], r, q) for sid, r, q in ov["recvs"]], "views": cvs}
            d = ov.get("dot")
            if d is not None:
                if d["x"] not in cidx or d["y"] not in cidx:
                    return
                plan["overlap"]["dot"] = dict(d, x=cidx[d["x"]], y=cidx[d["y"]])
        if rec.get("sdpub") is not None:
            plan["sdpub"] = rec["sdpub"]
        plan["views"], plan["fold"] = vs, fold
        dev = set()
        for item in vs:
            cv = item[0] if kp is None else item
            dev.update(c for _, c, _ in cv[1])
        for cv in plan.get("overlap", {}).get("views", ()):
            dev.update(c for _, c, _ in cv[1])
        for cv, *_ in fold:
            dev.update(c for _, c, _ in cv[1])
        plan["dev"] = sorted(dev)
        plan["ensure"] = sorted({(cidx[sid], rect) for sid, rect in rec["ensure"]})
        plan["inits"] = [(cidx[sid], rects) for sid, rects in rec["inits"]]
        x = rec["xfer"]
        if x is not None:
            n, xs, peers, dirs, los, his, nbytes = x
            if any(xs[i] not in cidx for i in range(n)):
                return
            x = (n, [cidx[xs[i]] for i in range(n)], peers, dirs, los, his, nbytes)
        plan["xfer"] = x
        plan["post"] = tuple((c, tuple(tuple(v) for v in self.stores[sid].valid), tuple(self.stores[sid].written))
                             for c, sid in enumerate(sids))
        if len(self._mplans) > 4096:
            self._mplans.clear()
        self._mplans[key] = plan

    @staticmethod
    def _rebind(cv, bases):
        views, patches = cv
        if patches and patches[0][0] is None:  # a single view
            nv = dk_view()
            ctypes.pointer(nv)[0] = views
            nv.ptr = bases[patches[0][1]] + patches[0][2]
            return nv
        nv = (dk_view * len(views))()
        ctypes.memmove(nv, views, ctypes.sizeof(views))
        for idx, c, off in patches:
            nv[idx].ptr = bases[c] + off
        return nv

    def _mplan_replay(self, hit, task, kp, sids, sd=None) -> None:
        recs = [self.rec(sid) for sid in sids]
        for c, rects in hit["inits"]:
            self._materialize_init(recs[c], rects)
        for c, rect in hit["ensure"]:
            self._ensure(recs[c], rect)
        for c in hit["dev"]:
            self._device(recs[c])
        bases = [r.base for r in recs]
        x = hit["xfer"]
        if x is not None:
            n, cs, peers, dirs, los, his, nbytes = x
            self._exchange(n, (c_int64 * n)(*[sids[c] for c in cs]), peers, dirs, los, his)
            self.stats.transfers += n
            self.stats.bytes_moved += nbytes
            if kp is not None:
                self.mark("halo_done")
        if kp is None and hit.get("overlap") is not None:
            ov = hit["overlap"]
            d = ov.get("dot")
            dot = None if d is None else (self._sd_regions(len(d["rows"])), d["rows"])
            self._issue_spmv_overlap([(sids[c], r, q) for c, r, q in ov["sends"]],
                                     [(sids[c], r, q) for c, r, q in ov["recvs"]],
                                     [self._rebind(cv, bases) for cv in ov["views"]], dot)
            self.stats.bytes_moved += sum(rg.volume(r) * recs[c].esize for c, r, _q in ov["recvs"] + ov["sends"])
            if d is not None:
                self._sd = {"x": sids[d["x"]], "y": sids[d["y"]],
                            "pts": {d["i"]: (d["yrect"], dot[0], runtime.SPMV_DOT_TOTAL, runtime.SPMV_DOT_DOUBLES,
                                             len(d["rows"]))}}
                self.spmv_dot_stats["spmv"] += 1
        elif kp is None:
            kind = task.kind.encode()
            for cv, n, wflags in hit["views"]:
                check(self.lib.dk_builtin(kind, self._rebind(cv, bases), n, wflags))
        else:
            h, _ = self.kernel_handle(kp)
            scal = self._scalars(task.scalars)
            ns, nsl = len(task.scalars), len(kp.slots)
            sp = hit.get("sdpub")
            if hit["pub"] and sp is not None:
                # the recorded window consumed the SpMV epilogue's p.q (Executor._run_kernel)
                epoch = self._p2p_epoch
                self._p2p_epoch += 1
                for sir, cv in enumerate(hit["views"]):
                    self._sd_publish(epoch, sir, sp["ridx"], sp["ntot"], sd["pts"][sp["pts"][sir]])
                    check(self.lib.dk_launch_pub_ex(sp["h"], self._rebind(cv, bases), nsl, scal, ns, epoch, sir,
                                                    1 if sp["ridx"] == 0 else 0, sp["ntot"]))
                self.spmv_dot_stats["consumed"] += 1
                self.spmv_dot_stats["replayed"] += 1
                self.mark("pub_done")
                self._p2p_fold(epoch, hit["counts"], [(self._rebind(cv, bases), first, stride, nv)
                                                      for cv, first, stride, nv in hit["fold"]])
                self.mark("wait_done")
                self.stats.p2p_folds += 1
            elif hit["pub"]:
                epoch = self._p2p_epoch
                self._p2p_epoch += 1
                for sir, cv in enumerate(hit["views"]):
                    check(self.lib.dk_launch_pub(h, self._rebind(cv, bases), nsl, scal, ns, epoch, sir))
                self.mark("pub_done")
                self._p2p_fold(epoch, hit["counts"], [(self._rebind(cv, bases), first, stride, nv)
                                                      for cv, first, stride, nv in hit["fold"]])
                self.mark("wait_done")
                self.stats.p2p_folds += 1
            else:
                for cv in hit["views"]:
                    check(self.lib.dk_launch(h, self._rebind(cv, bases), nsl, scal, ns, 0))
        for c, valid, written in hit["post"]:
            recs[c].valid = [list(v) for v in valid]
            recs[c].written = list(written)
        self.stats.launches += 1
        self.stats.points += len(hit["views"])
        self.stats.mplan_hits += 1

    def check_isolated(self, task: TaskDesc, temp_positions) -> None:
        """execute_isolated's claim checks (executor.py:236-262) on rects: a write
        overlapping another point's write, or a read / reduction touching cells
        another point writes, cannot run without communication."""
        pts = list(task.points())
        claims: dict[int, list] = {}
        for o, p in enumerate(pts):
            for j, a in enumerate(task.args):
                if j in temp_positions or not a.writes:
                    continue
                rect = rect_of(self.shape(a.store), a.part, p)
                if rg.empty(rect):
                    continue
                for o2, r2 in claims.get(a.store, ()):
                    if o2 != o and rg.overlaps(rect, r2):
                        raise ArenaViolation(f"write overlap on store {a.store} at point {p} of {task.kind}")
                claims.setdefault(a.store, []).append((o, rect))
        for o, p in enumerate(pts):
            for j, a in enumerate(task.args):
                if j in temp_positions or a.writes or a.store not in claims:
                    continue
                rect = rect_of(self.shape(a.store), a.part, p)
                if rg.empty(rect):
                    continue
                if any(o2 != o and rg.overlaps(rect, r2) for o2, r2 in claims[a.store]):
                    raise ArenaViolation(
                        f"point {p} of {task.kind} reads store {a.store} cells written by another point")

    def _execute_planned(self, task: TaskDesc, kp: KProg | None, temp_positions, pkey,
                         isolated: bool = False, spmv_dot=None) -> None:
        pts = list(task.points())
        V = len(pts)
        prank = [self.point_rank(i, V) for i in range(V)]
        rects = [[rect_of(self.shape(a.store), a.part, p) for a in task.args] for p in pts]
        for j, a in enumerate(task.args):
            if j not in temp_positions:
                self.rec(a.store)

        # access roles per argument
        if kp is None:
            # OPAQUE adds 1.0 to its W args in place (executor.py:101-104): it reads them
            reads = [a.reads or (a.writes and task.kind == "OPAQUE") for a in task.args]
            writes = [a.writes for a in task.args]
            reduces = [a.reduces for a in task.args]
        else:
            read_first, stored, red_slots = self._access(kp)
            reads = [False] * len(task.args)
            writes = [False] * len(task.args)
            reduces = [False] * len(task.args)
            for i, s in enumerate(kp.slots):
                if s.local:
                    continue
                a = task.args[s.arg]
                if i in read_first:
                    reads[s.arg] = True
                if i in stored and a.writes:
                    writes[s.arg] = True
                if i in red_slots:
                    reduces[s.arg] = True
        multi = self.world > 1

        # what each rank must hold before the launch
        need: dict[int, dict[int, list]] = {}
        for i in range(V):
            q = prank[i]
            for j, a in enumerate(task.args):
                if j in temp_positions:
                    continue
                rect = rects[i][j]
                if rg.empty(rect):
                    continue
                if reads[j]:
                    if kp is None and task.kind == "SPMV_CSR" and j == 3:
                        rect = self._csr_footprint(task, pts[i], rect)
                    need.setdefault(q, {}).setdefault(a.store, []).append(rect)
                if reduces[j]:
                    if multi and a.part.is_none:
                        for o in range(self.world):
                            need.setdefault(o, {}).setdefault(a.store, []).append(rect)
                    else:
                        need.setdefault(q, {}).setdefault(a.store, []).append(rect)
        if multi:
            self._check_cross_rank(task, prank, rects, reads, writes, temp_positions)
        overlap = kp is None and self._spmv_overlap_ok(task, prank)
        if overlap:
            # the x halo moves by copy engine while the interior rows run (_run_spmv_overlap)
            lay, own, halo_need = self._spmv_split(task, pts)
            for q in range(self.world):
                need[q][task.args[3].store] = [own[q]]
            self._satisfy(need)
            moves = self._satisfy(halo_need, defer=True)
        else:
            self._satisfy(need)
            if kp is not None:
                self.mark("halo_done")

        mine = [i for i in range(V) if prank[i] == self.rank]
        if overlap:
            self._run_spmv_overlap(task, pts, mine, rects, lay, moves)
        elif kp is None:
            self._run_builtin(task, pts, mine, rects, prank)
        else:
            recorded = self._run_kernel(task, kp, mine, prank, rects, temp_positions, reduces, isolated, spmv_dot)
            if recorded is not None and self.world == 1 and pkey is not None:
                # launch-plan cache: a memo-replayed window over the same
                # stores re-launches with the bound views as they are
                if len(self._plans) > 4096:
                    self._plans.clear()
                recs = tuple((a.store, self.stores[a.store]) for j, a in enumerate(task.args)
                             if j not in temp_positions)
                self._plans[pkey] = (kp, recs, recorded)
        self.stats.launches += 1
        self.stats.points += len(mine)

        # bookkeeping of the launch's effects (all ranks, all points)
        for i in range(V):
            for j, a in enumerate(task.args):
                if j in temp_positions:
                    continue
                if writes[j]:
                    self._wrote(a.store, rects[i][j], prank[i])
                if reduces[j] and not (multi and a.part.is_none):
                    self._wrote(a.store, rects[i][j], prank[i])
        if multi:
            for j, a in enumerate(task.args):
                if reduces[j] and a.part.is_none and j not in temp_positions:
                    r = self.stores[a.store]
                    for o in range(self.world):
                        r.valid[o] = rg.add(r.valid[o], r.full)
                    r.written = rg.add(r.written, r.full)

    # ------------------------------------------- SpMV with an overlapped halo
    # One tile per rank of the row-band Poisson matrix: rows [nx, t - nx) of a
    # tile reference only x rows the rank owns, so they run while the two
    # one-grid-row halos come in by copy engine (dk_dma_send on a side stream,
    # dk_dma_recv on the main stream after the interior rows); the boundary
    # rows follow.  Same kernels, same per-row order: bit-identical results.
    def _spmv_overlap_ok(self, task: TaskDesc, prank) -> bool:
        if not (self.world > 1 and self._p2p and task.kind == "SPMV_CSR"
                and os.environ.get("DK_OVERLAP_HALO", "1") == "1"):
            return False
        spec = self.init.get(task.args[1].store)
        if not spec or spec.get("kind") != "csr_cols" or int(spec["k"]) != len(prank):
            return False
        if list(prank) != list(range(self.world)) or task.launch != (self.world,):
            return False
        lay = poisson_tile_layout(int(spec["nx"]), int(spec["ny"]), int(spec["k"]))
        return lay["t"] > 2 * lay["nx"] and self.shape(task.args[3].store) == (lay["n"],) \
            and task.args[3].part.is_none

    def _spmv_split(self, task: TaskDesc, pts):
        spec = self.init[task.args[1].store]
        lay = poisson_tile_layout(int(spec["nx"]), int(spec["ny"]), int(spec["k"]))
        t, n = lay["t"], lay["n"]
        xs = task.args[3].store
        own = {q: ((q * t,), ((q + 1) * t,)) for q in range(self.world)}
        halo = {}
        for q in range(self.world):
            f = self._csr_footprint(task, pts[q], ((0,), (n,)))
            parts = [x for x in rg.minus([f], [own[q]]) if not rg.empty(x)]
            halo[q] = {xs: parts}
        return lay, own, halo

    def _run_spmv_overlap(self, task, pts, mine, rects, lay, moves) -> None:
        t, nx = lay["t"], lay["nx"]
        i = mine[0]
        recs = [self.stores[a.store] for a in task.args]
        for rec, rect in zip(recs, rects[i]):
            self._ensure(rec, rect)
        r_rp, r_cl, r_vl, r_x, r_y = recs
        rp0, y0 = rects[i][0][0][0], rects[i][4][0][0]

        def rows(a, b):
            views = (dk_view * 5)()
            views[0] = self.view(r_rp, ((rp0 + a,), (rp0 + b + 1,)))
            views[1] = self.view(r_cl, rects[i][1])
            views[2] = self.view(r_vl, rects[i][2])
            views[3] = self.view(r_x, r_x.full)
            views[4] = self.view(r_y, ((y0 + a,), (y0 + b,)))
            return views

        spans = [(a, b) for a, b in ((nx, t - nx), (0, nx), (t - nx, t)) if b > a]
        launches = [rows(a, b) for a, b in spans]
        sends = [(x[0], x[1], x[3]) for x in moves if x[2] == self.rank]
        recvs = [(x[0], x[1], x[2]) for x in moves if x[3] == self.rank]
        dot = None
        if self.fuse_spmv_dot and self.shape(task.args[3].store) == self.shape(task.args[4].store):
            # the partial-dot epilogue per row span, one buffer region (and one total) per span
            dot = (self._sd_regions(len(spans)), [y0 + a for a, _b in spans])
        if self._rec is not None:
            slots = [(j, a.store) for j, a in enumerate(task.args)]
            self._rec["overlap"] = {"sends": sends, "recvs": recvs, "views": [(v, slots) for v in launches]}
            if dot is not None:
                self._rec["overlap"]["dot"] = {"rows": dot[1], "i": i, "yrect": rects[i][4],
                                               "x": task.args[3].store, "y": task.args[4].store}
        self._issue_spmv_overlap(sends, recvs, launches, dot)
        if dot is not None:
            D = runtime.SPMV_DOT_DOUBLES
            self._sd = {"x": task.args[3].store, "y": task.args[4].store,
                        "pts": {i: (rects[i][4], dot[0], runtime.SPMV_DOT_TOTAL, D, len(spans))}}
            self.spmv_dot_stats["spmv"] += 1

    def _issue_spmv_overlap(self, sends, recvs, launches, dot=None) -> None:
        """Side stream: the halo sends (copy engine); main stream: the interior rows, the halo
        receives, the boundary rows.  ``sends`` / ``recvs``: (store, rect, peer).  ``dot``:
        (dk_spmv_csr_dot regions, first x row per launch) for the partial-dot epilogue."""

        def spmv(k, views):
            if dot is None:
                check(self.lib.dk_builtin(b"SPMV_CSR", views, 5, wflags))
                return
            np_ = c_int()
            check(self.lib.dk_spmv_csr_dot(views, dot[0] + 8 * runtime.SPMV_DOT_DOUBLES * k, dot[1][k], byref(np_)))

        def enc(lst):
            m = len(lst)
            sids = (c_int64 * max(m, 1))(*[x[0] for x in lst])
            peers = (c_int32 * max(m, 1))(*[x[2] for x in lst])
            los = (c_int64 * (4 * max(m, 1)))()
            his = (c_int64 * (4 * max(m, 1)))()
            for k, x in enumerate(lst):
                los[4 * k], his[4 * k] = x[1][0][0], x[1][1][0]
            return m, sids, peers, los, his

        main = self.stream()
        if self._side is None:
            s = c_uint64()
            check(self.lib.dk_stream_new(byref(s)))
            self._side = s.value
            evs = []
            for _ in range(2):
                e = c_uint64()
                check(self.lib.dk_event_new(byref(e)))
                evs.append(e.value)
            self._side_ev = evs
        if sends:
            check(self.lib.dk_event_record(self._side_ev[0]))  # p is final on the main stream here
            check(self.lib.dk_set_stream(self._side))
            try:
                check(self.lib.dk_stream_wait_event(self._side_ev[0]))
                check(self.lib.dk_dma_send(*enc(sends)))
                check(self.lib.dk_event_record(self._side_ev[1]))
            finally:
                check(self.lib.dk_set_stream(main))
        wflags = (c_int32 * 5)(0, 0, 0, 0, 1)
        spmv(0, launches[0])  # interior: own x rows only
        self.mark("interior_done")
        if recvs:
            check(self.lib.dk_dma_recv(*enc(recvs)))
        self.mark("halo_in")
        for k, views in enumerate(launches[1:], 1):
            spmv(k, views)
        if sends:
            check(self.lib.dk_stream_wait_event(self._side_ev[1]))  # p is not rewritten before the sends read it
        self.stats.p2p_halos += 1

    def _csr_footprint(self, task: TaskDesc, p, full):
        """Columns of x an SPMV_CSR tile actually reads (NonePart reads the whole store).

        For the Poisson tiles (init spec known on every rank) the referenced
        columns are the tile's rows +- one grid row; the coherence planner
        then moves a one-row halo instead of gathering all of x.  Unknown
        matrices keep the conservative whole-store footprint.
        """
        spec = self.init.get(task.args[1].store)
        if not spec or spec.get("kind") != "csr_cols":
            return full
        lay = poisson_tile_layout(int(spec["nx"]), int(spec["ny"]), int(spec["k"]))
        t, nx, n = lay["t"], lay["nx"], lay["n"]
        q = p[0]
        if full[1][0] != n:
            return full
        return ((max(0, q * t - nx),), (min(n, (q + 1) * t + nx),))

    def _access(self, kp: KProg):
        hit = self._acc.get(id(kp))
        if hit is None or hit[0] is not kp:
            hit = (kp, slot_access(kp))
            self._acc[id(kp)] = hit
        return hit[1]

    def _check_cross_rank(self, task, prank, rects, reads, writes, temp_positions) -> None:
        """Points of one launch on different GPUs must not need each other's data.

        The reference runs points in lexicographic order (executor.py:193-195),
        so point q observes an earlier point p's writes.  Running them
        concurrently on different GPUs is equivalent unless q reads -- before
        writing it itself -- a region an earlier point on another GPU writes.
        Overlapping writes alone are fine: the later point's value is the one
        the coherence bookkeeping keeps (``_wrote`` in point order).
        """
        V = len(prank)
        if len(set(prank)) < 2:
            return
        wr = [(i, prank[i], a.store, rects[i][j]) for i in range(V) for j, a in enumerate(task.args)
              if writes[j] and j not in temp_positions]
        if not wr:
            return
        for i in range(V):
            for j, a in enumerate(task.args):
                if j in temp_positions or not reads[j]:
                    continue
                for p, q, sid, w in wr:
                    if p < i and q != prank[i] and sid == a.store and rg.overlaps(w, rects[i][j]):
                        raise UnsupportedError(
                            f"{task.kind}: point {i} reads store {sid} written by point {p} on another GPU"
                        )

    def _alias_candidates(self, kp: KProg, task: TaskDesc) -> bool:
        """Does a stored slot share its store with another heap-bound slot?  (cached per binding)"""
        key = (id(kp), task.args)
        hit = self._alias_c.get(key)
        if hit is not None and hit[0] is kp:
            return hit[1]
        _, stored, _ = self._access(kp)
        params = [(i, task.args[s.arg].store) for i, s in enumerate(kp.slots) if not s.local]
        wstores = {sid for i, sid in params if i in stored}
        res = len(wstores) > 0 and sum(1 for _, sid in params if sid in wstores) > len(
            {i for i, sid in params if i in stored})
        if len(self._alias_c) > 4096:
            self._alias_c.clear()
        self._alias_c[key] = (kp, res)
        return res

    def _aliased(self, kp: KProg, task: TaskDesc, rects_p):
        """Aliasing plan of one point (aliasing.plan): rewritten kernel handle and copy-in slots."""
        store_of = {i: task.args[s.arg].store for i, s in enumerate(kp.slots) if not s.local}
        rects = {i: rects_p[kp.slots[i].arg] for i in store_of}
        mapping, copy_in = aliasing.plan(kp, store_of, rects)
        h = None
        if mapping:
            key = (id(kp), tuple(sorted(mapping.items())))
            hit = self._alias_k.get(key)
            if hit is None or hit[0] is not kp:
                hit = (kp, aliasing.rewrite(kp, mapping))
                self._alias_k[key] = hit
            h, _ = self.kernel_handle(hit[1])
        return h, copy_in

    def _copy_in(self, view: dk_view) -> tuple[dk_view, int]:
        """Copy a bound view into dense scratch (stream-ordered); returns (scratch view, pointer)."""
        if view.dtype != DK_F64:
            raise UnsupportedError("copy-in of an aliased non-f64 view")
        n = 1
        for d in range(view.rank):
            n *= view.ext[d]
        p = c_uint64()
        check(self.lib.dk_scratch_alloc(8 * max(n, 1), byref(p)))
        dst = dk_view()
        dst.ptr, dst.rank, dst.dtype = p.value, view.rank, DK_F64
        st_ = 1
        for d in range(view.rank - 1, -1, -1):
            dst.ext[d] = view.ext[d]
            dst.stride[d] = st_
            st_ *= max(view.ext[d], 1)
        if n:
            h, _ = self.kernel_handle(aliasing.copy_kprog(view.rank))
            pair = (dk_view * 2)(view, dst)
            check(self.lib.dk_launch(h, pair, 2, self._scalars(()), 0, 0))
        return dst, p.value

    def _spmv_dot_match(self, task, kp, mine, rects, sd):
        """The reduce statement ``t += sum(p * q)`` this window would compute from the SpMV's own
        x-tile and result (same rects), if any: (nest, stmt index, target slot)."""
        for n, (_dom, _rank, stmts) in enumerate(kp.nests):
            for k, st in enumerate(stmts):
                if st[0] != "reduce":
                    continue
                e = st[2]
                if e[0] != "bin" or e[1] != "*" or e[2][0] != "ld" or e[3][0] != "ld":
                    continue
                a, b = e[2][1], e[3][1]
                if kp.slots[a].local or kp.slots[b].local or any(e[2][2]) or any(e[3][2]):
                    continue
                sa, sb = task.args[kp.slots[a].arg].store, task.args[kp.slots[b].arg].store
                if {sa, sb} != {sd["x"], sd["y"]} or sa == sb:
                    continue
                if sum(1 for _, _, sts in kp.nests for t in sts if t[0] == "reduce" and t[1] == st[1]) != 1:
                    continue
                if len(stmts) < 2 or self.shape(task.args[kp.slots[st[1]].arg].store) != ():
                    continue
                if set(mine) != set(sd["pts"]):
                    continue
                if all(rects[i][kp.slots[a].arg] == sd["pts"][i][0] == rects[i][kp.slots[b].arg] for i in mine):
                    return n, k, st[1]
        return None

    def _run_kernel(self, task, kp, mine, prank, rects, temp_positions, reduces, isolated=False,
                    spmv_dot=None) -> None:
        if len(kp.scalar_names) != len(task.scalars):
            raise BackendError(
                f"task {task.kind} carries {len(task.scalars)} scalars, kernel expects {len(kp.scalar_names)}"
            )
        sd_fold = None
        sd_pub = None  # several GPUs: (position of p.q among the reductions, their count, original kernel)
        if spmv_dot is not None:
            m = self._spmv_dot_match(task, kp, mine, rects, spmv_dot)
            if m is not None:
                n, k, tslot = m
                order = [(n2, k2) for n2, (_d, _r, sts) in enumerate(kp.nests) for k2, st in enumerate(sts)
                         if st[0] == "reduce"]
                ridx = order.index((n, k))
                # several GPUs: the SpMV's per-point p.q total rides in the window's own board block,
                # which needs it first or last among the reductions (the kernel writes the rest)
                cnt = [0] * self.world
                for q in prank:
                    cnt[q] += 1
                ok = self.world == 1 or (self._p2p and not isolated and ridx in (0, len(order) - 1)
                                         and len(order) <= runtime.P2P_RED and min(cnt) >= 1
                                         and max(cnt) <= runtime.P2P_POINTS)
                if ok:
                    key = (id(kp), "spmv_dot", n, k)
                    hit = self._alias_k.get(key)
                    if hit is None or hit[0] is not kp:
                        nests = list(kp.nests)
                        dom, rank, stmts = nests[n]
                        nests[n] = (dom, rank, stmts[:k] + stmts[k + 1:])
                        hit = (kp, KProg(kp.slots, kp.scalar_names, kp.ntemps, tuple(nests), kp.fused_names))
                        self._alias_k[key] = hit
                    if self.world == 1:
                        sd_fold = (tslot, spmv_dot)
                    else:
                        sd_pub = (ridx, len(order), kp, spmv_dot)
                    kp = hit[1]
        h, nred = self.kernel_handle(kp)
        scal = self._scalars(task.scalars)
        nslots = len(kp.slots)
        red_kp = kp if sd_pub is None else sd_pub[2]
        red_targets = [
            (st[1], red_kp.slots[st[1]]) for _, _, stmts in red_kp.nests for st in stmts if st[0] == "reduce"
        ]
        use_totals = (self.world > 1 or isolated) and nred > 0
        V = len(prank)
        totals = 0
        maxp = 0
        pub_slot = -1  # reduction epoch of a peer-board launch (-1: none)
        if use_totals:
            counts = [0] * self.world
            for q in prank:
                counts[q] += 1
            maxp = max(counts)
            # the board ring is only safe when every rank publishes into every slot
            # it consumes: a rank without points would only read, so it could fall
            # DK_P2P_SLOTS epochs behind its peers (their publishes would overwrite
            # a slot it has not folded yet) -- such launches take the NCCL gather
            if self._p2p and not isolated and min(counts) >= 1 and maxp <= runtime.P2P_POINTS and nred <= runtime.P2P_RED:
                pub_slot = self._p2p_epoch  # the reduction epoch (board slot = epoch mod P2P_SLOTS)
                self._p2p_epoch += 1
                use_totals = False
        if sd_pub is not None and pub_slot < 0:
            raise BackendError("SpMV + partial-dot epilogue without the peer-board reduction path")
        if use_totals:
            nbytes = 8 * maxp * nred
            tb = c_uint64()
            check(self.lib.dk_scratch_alloc(nbytes * (self.world + 1), byref(tb)))
            totals = tb.value
            check(self.lib.dk_memset_zero(totals, nbytes * (self.world + 1)))
        has_local = any(s.local for s in kp.slots)
        recorded = [] if not (use_totals or has_local or pub_slot >= 0) else None
        if self._rec is not None:
            if use_totals or has_local:
                self._rec["ok"] = False
            elif pub_slot >= 0:
                self._rec["pub"] = True
                self._rec["counts"] = (c_int32 * self.world)(*counts)
        aliased = self._alias_candidates(kp, task)
        if sd_fold is not None or sd_pub is not None:
            recorded = None
            if self._rec is not None:
                if sd_pub is not None and pub_slot >= 0 and not aliased:
                    self._rec["sdpub"] = {"ridx": sd_pub[0], "ntot": sd_pub[1], "h": h, "pts": list(mine)}
                else:
                    self._rec["ok"] = False
        if aliased:
            recorded = None  # copy-ins and rewritten kernels are planned per launch
            if self._rec is not None:
                self._rec["ok"] = False
        for slot_in_rank, i in enumerate(mine):
            views = (dk_view * nslots)()
            rp = rects[i]
            h_pt, copy_in = self._aliased(kp, task, rp) if aliased else (None, [])
            scratch = []
            for si, s in enumerate(kp.slots):
                rect = rp[s.arg]
                if s.local:
                    ext = tuple(max(0, h2 - l) for l, h2 in zip(*rect))
                    n = 1
                    for e in ext:
                        n *= e
                    p = c_uint64()
                    check(self.lib.dk_scratch_alloc(8 * max(n, 1), byref(p)))
                    check(self.lib.dk_memset_zero(p.value, 8 * max(n, 1)))
                    scratch.append(p.value)
                    v = views[si]
                    v.ptr = p.value
                    v.rank = len(ext)
                    v.dtype = DK_F64
                    st_ = 1
                    for d in range(len(ext) - 1, -1, -1):
                        v.ext[d] = ext[d]
                        v.stride[d] = st_
                        st_ *= max(ext[d], 1)
                else:
                    r = self.stores[task.args[s.arg].store]
                    self._ensure(r, rect)
                    views[si] = self.view(r, rect)
            for si in copy_in:
                views[si], p = self._copy_in(views[si])
                scratch.append(p)
            hl = h if h_pt is None else h_pt
            if sd_pub is not None:
                # the point's p.q total (its SpMV partials folded in order) goes into its board
                # block first; the window kernel writes its own totals beside it and publishes all
                ridx, ntot, _kp0, sd = sd_pub
                self._sd_publish(pub_slot, slot_in_rank, ridx, ntot, sd["pts"][i])
                check(self.lib.dk_launch_pub_ex(hl, views, nslots, scal, len(task.scalars), pub_slot, slot_in_rank,
                                                1 if ridx == 0 else 0, ntot))
            elif pub_slot >= 0:
                check(self.lib.dk_launch_pub(hl, views, nslots, scal, len(task.scalars), pub_slot, slot_in_rank))
            else:
                tot = totals + 8 * nred * (self.rank * maxp + slot_in_rank) if use_totals else 0
                check(self.lib.dk_launch(hl, views, nslots, scal, len(task.scalars), tot))
            for p in scratch:
                check(self.lib.dk_scratch_free(p))
            if recorded is not None:
                recorded.append(views)
            if self._rec is not None:
                self._rec["views"].append((views, [
                    (si, task.args[s.arg].store) for si, s in enumerate(kp.slots) if not s.local]))
        if sd_fold is not None:
            # the removed statement's p.q: each point's SpMV partials folded in a fixed order into
            # a total, then target += total in point order (executor.py:193-195)
            tslot, sd = sd_fold
            a = task.args[kp.slots[tslot].arg]
            r = self.stores[a.store]
            for i in sorted(mine):
                _rect, parts, first, stride, nt = sd["pts"][i]
                tv = self.view(r, rects[i][kp.slots[tslot].arg])
                if nt == 1:
                    check(self.lib.dk_accum(byref(tv), parts, first, stride, 1))
                    continue
                # several row spans: their totals folded first, then added (one total per point)
                tot = c_uint64()
                check(self.lib.dk_scratch_alloc(8, byref(tot)))
                tv0 = dk_view()
                tv0.ptr, tv0.rank, tv0.dtype = tot.value, 0, DK_F64
                check(self.lib.dk_memset_zero(tot.value, 8))
                check(self.lib.dk_accum(byref(tv0), parts, first, stride, nt))
                check(self.lib.dk_accum(byref(tv), tot.value, 0, 1, 1))
                check(self.lib.dk_scratch_free(tot.value))
            self.spmv_dot_stats["consumed"] += 1
        if use_totals:
            block = maxp * nred
            gathered = totals + 8 * block  # [world][maxp][nred] after the allgather
            if self.world > 1:
                check(self.lib.dk_comm_allgather_f64(totals + 8 * block * self.rank, gathered, block))
            else:
                gathered = totals
            if isolated:
                self._fold_isolated(task, prank, rects, red_targets, gathered, maxp, nred)
            else:
                self._fold(task, kp, prank, rects, red_targets, gathered, maxp, nred)
            check(self.lib.dk_scratch_free(totals))
        elif pub_slot >= 0:
            self.mark("pub_done")
            ops = []
            self._collect = ops
            try:
                self._fold(task, red_kp, prank, rects, red_targets, 0, runtime.P2P_POINTS, len(red_targets))
            finally:
                self._collect = None
            if sd_pub is not None:
                self.spmv_dot_stats["consumed"] += 1
            self._p2p_fold(pub_slot, (c_int32 * self.world)(*counts), ops)
            self.mark("wait_done")
            self.stats.p2p_folds += 1
        return recorded

    def _sd_publish(self, epoch, point, ridx, ntot, pt) -> None:
        """The point's p.q total (its SpMV row spans' totals folded in order) into its board
        block at statement position ``ridx``, before the window kernel publishes the block."""
        _rect, parts, first, stride, nt = pt
        blk = c_uint64()
        check(self.lib.dk_p2p_block(epoch, point, ntot, byref(blk)))
        pv = dk_view()
        pv.ptr, pv.rank, pv.dtype = blk.value + 8 * ridx, 0, DK_F64
        check(self.lib.dk_memset_zero(pv.ptr, 8))
        check(self.lib.dk_accum(byref(pv), parts, first, stride, nt))

    def _accum(self, sid, tv, gathered, first, stride, n) -> None:
        if self._collect is not None:
            self._collect.append((tv, first, stride, n))
        else:
            check(self.lib.dk_accum(byref(tv), gathered, first, stride, n))
        if self._rec is not None:
            self._rec["fold"].append(((tv, [(None, sid)]), first, stride, n))

    def _p2p_fold(self, epoch: int, counts, ops) -> None:
        """Wait for the board slot of ``epoch`` and apply the fold ops in order: one kernel
        (dk_p2p_wait_fold) when every target is a scalar, else the wait then dk_accum per op."""
        if len(ops) <= runtime.P2P_FOLDS and all(tv.rank == 0 for tv, *_ in ops):
            n = len(ops)
            check(self.lib.dk_p2p_wait_fold(
                epoch, counts, n, (c_uint64 * max(n, 1))(*[tv.ptr for tv, *_ in ops]),
                (c_int64 * max(n, 1))(*[o[1] for o in ops]), (c_int64 * max(n, 1))(*[o[2] for o in ops]),
                (c_int32 * max(n, 1))(*[o[3] for o in ops])))
            return
        g = c_uint64()
        check(self.lib.dk_p2p_wait(epoch, counts, byref(g)))
        for tv, first, stride, n in ops:
            check(self.lib.dk_accum(byref(tv), g.value, first, stride, n))

    def _fold(self, task, kp, prank, rects, red_targets, gathered, maxp, nred) -> None:
        """Fold gathered per-point totals ([world][maxp][nred]) in lexicographic point order."""
        V = len(prank)
        slot_of_point = []
        seen = [0] * self.world
        for q in prank:
            slot_of_point.append(seen[q])
            seen[q] += 1
        idx = [[(prank[i] * maxp + slot_of_point[i]) * nred + k for k in range(nred)] for i in range(V)]
        tslots = [sl for sl, _ in red_targets]
        distinct = len(set(tslots)) == len(tslots)
        if distinct:
            for k, (sl, s) in enumerate(red_targets):
                a = task.args[s.arg]
                if a.part.is_none:
                    r = self.stores[a.store]
                    self._ensure(r, r.full)
                    tv = self.view(r, r.full)
                    ks = [idx[i][k] for i in range(V)]
                    stride = ks[1] - ks[0] if V > 1 else 1
                    if all(ks[t] == ks[0] + t * stride for t in range(V)):
                        self._accum(a.store, tv, gathered, ks[0], stride, V)
                    else:
                        for kk in ks:
                            self._accum(a.store, tv, gathered, kk, 1, 1)
                else:
                    for i in range(V):
                        if prank[i] != self.rank:
                            continue
                        r = self.stores[a.store]
                        tv = self.view(r, rects[i][s.arg])
                        self._accum(a.store, tv, gathered, idx[i][k], 1, 1)
            return
        for i in range(V):
            for k, (sl, s) in enumerate(red_targets):
                a = task.args[s.arg]
                if not a.part.is_none and prank[i] != self.rank:
                    continue
                r = self.stores[a.store]
                rect = r.full if a.part.is_none else rects[i][s.arg]
                self._ensure(r, rect)
                tv = self.view(r, rect)
                self._accum(a.store, tv, gathered, idx[i][k], 1, 1)

    def _fold_isolated(self, task, prank, rects, red_targets, gathered, maxp, nred) -> None:
        """execute_isolated's combine (executor.py:280-293): per point, a zeroed arena per
        reduction target collects that target's statements in order, then
        ``dest += arena`` in point order."""
        V = len(prank)
        seen = [0] * self.world
        arena = c_uint64()
        check(self.lib.dk_scratch_alloc(8, byref(arena)))
        av = dk_view()
        av.ptr, av.rank, av.dtype = arena.value, 0, DK_F64
        groups: dict[int, list[int]] = {}
        for k, (sl, _s) in enumerate(red_targets):
            groups.setdefault(sl, []).append(k)
        for i in range(V):
            q = prank[i]
            base = (q * maxp + seen[q]) * nred
            seen[q] += 1
            for sl, ks in groups.items():
                a = task.args[red_targets[ks[0]][1].arg]
                if not a.part.is_none and q != self.rank:
                    continue
                r = self.stores[a.store]
                rect = r.full if a.part.is_none else rects[i][red_targets[ks[0]][1].arg]
                self._ensure(r, rect)
                check(self.lib.dk_memset_zero(arena.value, 8))
                for k in ks:
                    check(self.lib.dk_accum(byref(av), gathered, base + k, 1, 1))
                tv = self.view(r, rect)
                check(self.lib.dk_accum(byref(tv), arena.value, 0, 1, 1))
        check(self.lib.dk_scratch_free(arena.value))

    def _run_builtin(self, task, pts, mine, rects, prank) -> None:
        n = len(task.args)
        wflags = (c_int32 * max(n, 1))(*[1 if a.writes else 0 for a in task.args])
        kind = task.kind.encode()
        red = [j for j, a in enumerate(task.args) if a.reduces]
        arenas = self.world > 1 and bool(red)
        if arenas and self._rec is not None:
            self._rec["ok"] = False
        if arenas:
            # per-point zero arenas for the Rd args (executor.py:280-281), then the
            # same allgather + point-order fold as kernel reductions
            for j in red:
                a = task.args[j]
                if not a.part.is_none or self.shape(a.store) != ():
                    raise UnsupportedError(f"{task.kind}: multi-GPU builtin reductions need rank-0 NonePart targets")
            counts = [0] * self.world
            for q in prank:
                counts[q] += 1
            maxp, nred = max(counts), len(red)
            block = maxp * nred
            tb = c_uint64()
            check(self.lib.dk_scratch_alloc(8 * block * (self.world + 1), byref(tb)))
            check(self.lib.dk_memset_zero(tb.value, 8 * block * (self.world + 1)))
        sd_pts = {}
        sd_base = 0
        # several GPUs: the consuming window can only carry p.q through its peer-board block
        # when every rank owns a point (Executor._run_kernel)
        sd_ok = self.world == 1 or (self._p2p and len(set(prank)) == self.world)
        for slot_in_rank, i in enumerate(mine):
            views = (dk_view * max(n, 1))()
            for j, a in enumerate(task.args):
                if arenas and j in red:
                    v = dk_view()
                    v.ptr = tb.value + 8 * (block * self.rank + slot_in_rank * nred + red.index(j))
                    v.rank, v.dtype = 0, DK_F64
                    views[j] = v
                    continue
                r = self.stores[a.store]
                self._ensure(r, rects[i][j])
                views[j] = self.view(r, rects[i][j])
            # numpy evaluates a builtin's result before assigning it (bufs["a2"][...] = a0 @ a1,
            # executor.py:93-94): an input overlapping a written argument is read from a copy
            scratch = []
            for j, a in enumerate(task.args):
                if not a.reads or a.writes:
                    continue
                if any(b.writes and b.store == a.store and k != j and rg.overlaps(rects[i][j], rects[i][k])
                       for k, b in enumerate(task.args)):
                    views[j], p = self._copy_in(views[j])
                    scratch.append(p)
            if scratch and self._rec is not None:
                self._rec["ok"] = False
            if (self.fuse_spmv_dot and task.kind == "SPMV_CSR" and not scratch and not arenas and sd_ok
                    and len(rects[i][4][0]) == 1 and self.shape(task.args[3].store) == self.shape(task.args[4].store)):
                # opt-in epilogue: the SpMV also emits x_tile . y (per-CTA partials folded by its
                # last CTA) for the next window; one buffer region per point
                if not sd_base:
                    sd_base = self._sd_regions(len(mine))
                reg = sd_base + 8 * runtime.SPMV_DOT_DOUBLES * slot_in_rank
                np_ = c_int()
                check(self.lib.dk_spmv_csr_dot(views, reg, rects[i][4][0][0], byref(np_)))
                sd_pts[i] = (rects[i][4], reg, runtime.SPMV_DOT_TOTAL, 1, 1)
                if self._rec is not None:
                    self._rec["ok"] = False
            else:
                check(self.lib.dk_builtin(kind, views, n, wflags))
            for p in scratch:
                check(self.lib.dk_scratch_free(p))
            if self._rec is not None:
                self._rec["views"].append(((views, [(j, a.store) for j, a in enumerate(task.args)]), n, wflags))
        if sd_pts:
            self._sd = {"x": task.args[3].store, "y": task.args[4].store, "pts": sd_pts}
            self.spmv_dot_stats["spmv"] += 1
        if arenas:
            gathered = tb.value + 8 * block
            check(self.lib.dk_comm_allgather_f64(tb.value + 8 * block * self.rank, gathered, block))
            seen = [0] * self.world
            order = []
            for q in prank:
                order.append((q, seen[q]))
                seen[q] += 1
            for i, (q, s) in enumerate(order):
                for k, j in enumerate(red):
                    r = self.stores[task.args[j].store]
                    self._ensure(r, r.full)
                    tv = self.view(r, r.full)
                    check(self.lib.dk_accum(byref(tv), gathered, (q * maxp + s) * nred + k, 1, 1))
            check(self.lib.dk_scratch_free(tb.value))

    # ---------------------------------------------------------- host access
    def upload(self, sid: int, host: np.ndarray) -> None:
        """Replace the whole store with ``host`` (every rank holds it valid)."""
        self.drain()
        r = self.rec(sid)
        np_dtype = np.float64 if r.dtype == "f64" else np.int32
        a = np.asarray(host, dtype=np_dtype)  # (ascontiguousarray would turn 0-d into (1,))
        if not a.flags.c_contiguous:
            a = a.copy(order="C")
        if a.shape != r.shape:
            raise ValueError(f"store {sid} has shape {r.shape}, got {a.shape}")
        self._ensure(r, r.full)
        check(self.lib.dk_store_upload_rect(sid, i64s(r.full[0]), i64s(r.full[1]), a.ctypes.data))
        check(self.lib.dk_sync())
        for o in range(self.world):
            r.valid[o] = [r.full]
        r.written = [r.full]

    def upload_async(self, sid: int, host: np.ndarray, rect=None) -> None:
        """Enqueue an H2D copy of ``rect`` from a full-store host array (pinned for overlap)."""
        self.drain()
        r = self.rec(sid)
        rect = rect or r.full
        self._ensure(r, rect)
        check(self.lib.dk_store_upload_rect(sid, i64s(rect[0]), i64s(rect[1]), host.ctypes.data))
        self._wrote(sid, rect, self.rank)

    def download(self, sid: int, out: np.ndarray | None = None, rect=None) -> np.ndarray | None:
        """Collective on all ranks: gather ``rect`` of the store to rank 0 and copy it out."""
        self.drain()
        r = self.rec(sid)
        rect = rect or r.full
        self._satisfy({0: {sid: [rect]}})
        if self.rank != 0:
            return None
        np_dtype = np.float64 if r.dtype == "f64" else np.int32
        if out is None:
            out = np.empty(r.shape, dtype=np_dtype)
        self._ensure(r, rect)
        check(self.lib.dk_store_download_rect(sid, i64s(rect[0]), i64s(rect[1]), out.ctypes.data))
        return out

    def download_local(self, sid: int, out: np.ndarray, rect) -> np.ndarray:
        """D2H of a rect this rank holds valid (no gather; ``out`` is full-store shaped)."""
        self.drain()
        r = self.rec(sid)
        if not rg.covered(r.valid[self.rank], rect):
            raise BackendError(f"store {sid} rect {rect} is not valid on rank {self.rank}")
        check(self.lib.dk_store_download_rect(sid, i64s(rect[0]), i64s(rect[1]), out.ctypes.data))
        return out

    def get(self, sid: int) -> np.ndarray | None:
        a = self.download(sid)
        if a is None:
            return None
        return a.astype(np.float64) if a.dtype != np.float64 else a

    def sync(self) -> None:
        self.drain()
        check(self.lib.dk_sync())

    def jit_stats(self) -> dict:
        m, c, d = c_int64(), c_int64(), c_int64()
        s = c_double()
        check(self.lib.dk_jit_stats(byref(m), byref(c), byref(d), byref(s)))
        return {"modules": m.value, "nvrtc_compiles": c.value, "disk_cache_hits": d.value,
                "nvrtc_seconds": round(s.value, 3)}

    def launch_count(self) -> int:
        n = c_int64()
        check(self.lib.dk_launch_count(byref(n)))
        return n.value

    def capture(self, fn) -> int:
        """Run ``fn()`` (enqueue-only executor calls, e.g. one memo-replayed iteration whose
        launches are already planned) under stream capture; returns a graph handle for
        :meth:`graph_launch`.  Any synchronising call inside ``fn`` fails the capture."""
        if self._pending:
            raise BackendError("capture() with a deferred launch segment pending (call drain() first)")
        check(self.lib.dk_graph_begin())
        g = c_uint64()
        try:
            fn()
        finally:
            rc = self.lib.dk_graph_end(byref(g))
        check(rc)
        return g.value

    def graph_launch(self, graph: int) -> None:
        check(self.lib.dk_graph_launch(c_uint64(graph)))

    def graph_destroy(self, graph: int) -> None:
        check(self.lib.dk_graph_destroy(c_uint64(graph)))

    def stream(self) -> int:
        s = c_uint64()
        check(self.lib.dk_get_stream(byref(s)))
        return s.value

    def set_stream(self, ptr: int) -> None:
        check(self.lib.dk_set_stream(ptr))


def replay(ex: Executor, events, on_free=True) -> None:
    """Drive the executor with recorded plan events (plan.PlanTrace.events)."""
    for kind, ev in events:
        if kind == "exec":
            ex.execute(ev.task, ev.kernel, ev.temp_positions)
        elif kind == "free" and on_free:
            ex.free(ev)
