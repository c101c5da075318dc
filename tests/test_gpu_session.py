"""Drop-in check: ``GpuSession`` is a ``diffusekit.Session`` whose execution runs on the B200.

Needs the reference front end importable (``baseline/_ref`` travels with the
repo snapshot; skipped otherwise).  The same event stream runs through the
unchanged reference ``Session`` (numpy executor) and through ``GpuSession``;
reports (fusion plan) must be identical and heaps equal.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REPO, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dk():
    for cand in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "diffusekit")):
            sys.dont_write_bytecode = True
            sys.path.insert(0, cand)
            import diffusekit

            return diffusekit
    pytest.skip("reference front end (diffusekit) not installed")


def _run(session, events, dk):
    from diffusekit.pipeline import run_events

    return run_events(session, events)


@pytest.mark.parametrize(
    "name,kw,cfg",
    [
        ("stencil", dict(size=34, nodes=2, iters=4), {}),
        ("stencil", dict(size=34, nodes=2, iters=3), {"fusion": False}),
        ("blackscholes_chain", dict(size=4096, nodes=4, iters=5), {}),
        ("jacobi", dict(size=16, nodes=4, iters=3), {}),
        ("cg_like", dict(size=16, nodes=4, iters=4), {}),
        ("cg_like", dict(size=16, nodes=4, iters=3), {"window": 2}),
    ],
)
def test_gpu_session_matches_reference_session(dk, name, kw, cfg):
    from diffusekit.pipeline import Session, SessionConfig
    from diffusekit.trace import gen_benchmark

    from paper_2406_18109_b200.session import GpuSession

    ref = Session(SessionConfig(**cfg))
    rep_ref = _run(ref, gen_benchmark(name, **kw), dk)
    gpu = GpuSession(SessionConfig(**cfg), device=0)
    try:
        rep_gpu = _run(gpu, gen_benchmark(name, **kw), dk)
        assert rep_gpu.fused_prefixes == rep_ref.fused_prefixes
        assert rep_gpu.temporaries_eliminated == rep_ref.temporaries_eliminated
        assert rep_gpu.loads == rep_ref.loads and rep_gpu.stores == rep_ref.stores
        assert [fr.kernel_stats for fr in rep_gpu.per_flush] == [fr.kernel_stats for fr in rep_ref.per_flush]
        for s in ref.live_store_ids():
            a, b = gpu.heap.get(s), ref.heap.get(s)
            if not same_bits(a, b):
                np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12 * max(1.0, float(np.abs(b).max())))
        if name == "blackscholes_chain" and not cfg:
            # memo-replayed steady iterations were relaunched as captured CUDA graphs (f3)
            gs = gpu.executor.graph_stats
            assert gs["captures"] >= 1 and gs["graph_launches"] >= 1, gs
    finally:
        gpu.executor.close()


def test_temporaries_never_reach_the_device(dk):
    """test_pipeline.py:42-54 on the GPU heap: only grid and work materialise."""
    from diffusekit.pipeline import SessionConfig
    from diffusekit.trace import gen_benchmark

    from paper_2406_18109_b200.session import GpuSession

    s = GpuSession(SessionConfig(), device=0)
    try:
        _run(s, gen_benchmark("stencil", iters=3), dk)
        assert set(s.executor.stores) == {0, 1}
    finally:
        s.executor.close()


def test_reference_exceptions(dk):
    from diffusekit.executor import UnknownTaskKindError
    from diffusekit.ir import Domain, IndexTask, Privilege, ProjectionFn, StoreArg, Tiling
    from diffusekit.pipeline import SessionConfig

    from paper_2406_18109_b200.session import GpuSession

    s = GpuSession(SessionConfig(), device=0)
    try:
        s.create_store(0, (4,))
        t = Tiling((2,), (0,), ProjectionFn.identity(1))
        s.submit(IndexTask("MYSTERY", Domain((2,)), (StoreArg(0, t, Privilege.WRITE),)))
        with pytest.raises(UnknownTaskKindError):
            s.flush()
    finally:
        s.executor.close()


def test_heap_arrays_injection(dk):
    """DOT accumulates onto injected contents (test_executor.py:85-96) through GpuHeap.arrays."""
    from diffusekit.ir import Domain, IndexTask, NonePart, Privilege, ProjectionFn, StoreArg, Tiling
    from diffusekit.pipeline import SessionConfig

    from paper_2406_18109_b200.session import GpuSession

    s = GpuSession(SessionConfig(), device=0)
    try:
        for sid, shp in ((0, (8,)), (1, (8,)), (2, ())):
            s.create_store(sid, shp)
        s.heap.arrays[0] = np.ones(8)
        s.heap.arrays[1] = np.ones(8)
        s.heap.arrays[2] = np.zeros(())
        p = Tiling((2,), (0,), ProjectionFn.identity(1))
        dot = IndexTask("DOT", Domain((4,)), (StoreArg(0, p, Privilege.READ), StoreArg(1, p, Privilege.READ),
                                              StoreArg(2, NonePart(), Privilege.REDUCE)))
        s.submit(dot)
        s.flush()
        assert s.heap.get(2)[()] == 8.0
        s.submit(dot)
        s.flush()
        assert s.heap.get(2)[()] == 16.0
    finally:
        s.executor.close()


def test_host_streamed_iterations(dk):
    """The e2e path: pinned x, y assigned through heap.arrays, the window reading them runs
    host-streamed (chunked H2D / kernel / D2H of stream_out(out)), results equal the reference
    Session's on the same inputs every iteration."""
    from diffusekit.pipeline import Session, SessionConfig, task_from_event
    from diffusekit.trace import CreatePartition, CreateStore, DropRef, Flush, TaskEvent, gen_blackscholes_chain, \
        partition_from_event

    from paper_2406_18109_b200.session import GpuSession

    n = 1 << 20
    its, cur = [], []
    for e in gen_blackscholes_chain(size=n, nodes=1, iters=6):
        cur.append(e)
        if isinstance(e, Flush):
            its.append(cur)
            cur = []

    def feed(sess, evs):
        for e in evs:
            if isinstance(e, CreateStore):
                sess.create_store(e.id, e.shape)
            elif isinstance(e, CreatePartition):
                sess.create_partition(e.id, partition_from_event(e))
            elif isinstance(e, TaskEvent):
                sess.submit(task_from_event(sess, e))
            elif isinstance(e, DropRef):
                sess.drop_ref(e.store)
            else:
                sess.flush()

    s = GpuSession(SessionConfig(), device=0)
    ref = Session(SessionConfig())
    try:
        hx, hy, ho = s.pinned((n,)), s.pinned((n,)), s.pinned((n,))
        s.stream_out(2, ho)
        rng = np.random.default_rng(3)
        for k, it in enumerate(its):
            head = [e for e in it if isinstance(e, (CreateStore, CreatePartition))]
            body = [e for e in it if not isinstance(e, (CreateStore, CreatePartition))]
            feed(s, head)
            feed(ref, head)
            hx[:] = rng.integers(1, 10, n)
            hy[:] = rng.random(n)
            s.heap.arrays[0] = hx
            s.heap.arrays[1] = hy
            ref.heap.arrays[0] = hx.copy()
            ref.heap.arrays[1] = hy.copy()
            feed(s, body)
            feed(ref, body)
            assert s.heap.get(2, out=ho) is ho
            assert same_bits(ho, ref.heap.get(2)), k
        assert s.streamed_windows >= len(its)
    finally:
        s.close()
