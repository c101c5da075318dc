"""Aliased arguments, POW and isolated execution against the reference (CPU).

``tests/golden/alias_streams.json.gz`` holds streams the UNCHANGED reference
ran (``make_alias_golden.py``): tasks that read and write one store through
several views, POW tasks, and ``SessionConfig(isolated=True)`` runs, some of
which the reference rejects with ``ArenaViolationError``.

* the oracle reproduces every heap byte-for-byte (pins the oracle on them);
* the executor, driven through the CPU stand-in in its *device model* (each
  kernel slot reads a private copy of its view, as a GPU thread does), must
  also reproduce them: that only holds if the identical-view rewrite and the
  copy-ins of ``aliasing.plan`` are right;
* isolated cases the reference rejects raise ``ArenaViolation`` at the same
  window.
"""

import numpy as np
import pytest

from conftest import golden_arrays, load_golden, same_bits


@pytest.fixture(scope="module")
def cases():
    return load_golden("alias_streams.json.gz")


def test_corpus_shape(cases):
    names = {c["name"] for c in cases}
    assert "alias_same_view/unfused" in names and "pow_integer/fused" in names
    assert sum(1 for c in cases if "error" in c) >= 10
    assert len(cases) >= 300


def test_oracle_matches_reference(cases):
    from oracle.interp import replay
    from paper_2406_18109_b200.plan import PlanTrace

    n = 0
    for c in cases:
        if "error" in c:
            continue
        tr = PlanTrace.from_json(c["trace"])
        heap = replay(tr)
        for s, want in golden_arrays(c).items():
            assert same_bits(heap.get(s), want), (c["name"], s)
        n += 1
    assert n > 250


def _executor_replay(tr, isolated, device_model=True):
    from fakedev import FakeLib
    from paper_2406_18109_b200.executor import Executor

    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes,
                  lib=FakeLib(0, 1, device_model=device_model))
    for kind, ev in tr.events:
        if kind == "exec":
            ex.execute(ev.task, ev.kernel, ev.temp_positions, isolated=isolated and ev.f > 1)
        elif kind == "free":
            ex.free(ev)
    return ex


def test_executor_device_model_matches_reference(cases):
    from paper_2406_18109_b200.errors import ArenaViolation
    from paper_2406_18109_b200.plan import PlanTrace

    checked = raised = 0
    for c in cases:
        tr = PlanTrace.from_json(c["trace"])
        iso = bool(tr.meta.get("isolated"))
        if "error" in c:
            with pytest.raises(ArenaViolation):
                _executor_replay(tr, iso)
            raised += 1
            continue
        ex = _executor_replay(tr, iso)
        for s, want in golden_arrays(c).items():
            assert same_bits(ex.get(s), want), (c["name"], s)
        checked += 1
    assert checked > 250 and raised >= 10


def test_device_model_detects_unhandled_aliasing(cases, monkeypatch):
    """Without the rewrite / copy-in the device model must produce wrong heaps
    (so the test above really exercises them)."""
    from paper_2406_18109_b200 import aliasing
    from paper_2406_18109_b200.plan import PlanTrace

    monkeypatch.setattr(aliasing, "plan", lambda kp, so, rects: (None, []))
    wrong = 0
    for c in cases:
        if "error" in c or c["name"].endswith("/isolated"):
            continue
        tr = PlanTrace.from_json(c["trace"])
        try:
            ex = _executor_replay(tr, False)
        except Exception:  # noqa: BLE001
            wrong += 1
            continue
        if any(not same_bits(ex.get(s), w) for s, w in golden_arrays(c).items()):
            wrong += 1
    assert wrong >= 10


def test_alias_plan_classification():
    from paper_2406_18109_b200 import aliasing
    from paper_2406_18109_b200.errors import UnsupportedError
    from paper_2406_18109_b200.ir import KProg, Slot

    def kp(stmts, nslots=3):
        return KProg(tuple(Slot(f"a{i}", i, False, "W" if i == nslots - 1 else "R", 1) for i in range(nslots)), (),
                     4, ((nslots - 1, 1, tuple(stmts)),), False)

    add = kp([("store", 2, (0,), ("bin", "+", ("ld", 0, (0,)), ("ld", 1, (0,))))])
    same = {0: ((0,), (4,)), 1: ((0,), (4,)), 2: ((0,), (4,))}
    m, ci = aliasing.plan(add, {0: 7, 1: 8, 2: 7}, same)
    assert m == {0: 2} and ci == []
    shifted = {0: ((0,), (4,)), 1: ((0,), (4,)), 2: ((2,), (6,))}
    m, ci = aliasing.plan(add, {0: 7, 1: 8, 2: 7}, shifted)
    assert m is None and ci == [0]
    disjoint = {0: ((0,), (4,)), 1: ((0,), (4,)), 2: ((4,), (8,))}
    assert aliasing.plan(add, {0: 7, 1: 8, 2: 7}, disjoint) == (None, [])
    # a read of the shifted view AFTER the overlapping store: numpy sees the new values
    late = kp([("store", 2, (0,), ("ld", 1, (0,))), ("store", 2, (0,), ("bin", "+", ("ld", 0, (0,)), ("ld", 2, (0,))))])
    with pytest.raises(UnsupportedError):
        aliasing.plan(late, {0: 7, 1: 8, 2: 7}, shifted)
    # overlap inside a per-element nest with offsets (sequential numpy loop)
    offs = kp([("store", 2, (0,), ("ld", 0, (1,)))])
    with pytest.raises(UnsupportedError):
        aliasing.plan(offs, {0: 7, 1: 8, 2: 7}, shifted)


def test_rewrite_preserves_numpy_semantics():
    """interpret(rewrite(kp)) with private copies per slot == interpret(kp) over aliased views."""
    from oracle.interp import interpret
    from paper_2406_18109_b200 import aliasing
    from paper_2406_18109_b200.ir import KProg, Slot

    slots = (Slot("b0", 0, False, "R", 1), Slot("b1", 1, False, "R", 1), Slot("b2", 2, False, "W", 1),
             Slot("b3", 3, False, "W", 1))
    # b2 = b0 + b1 ; b3 = b0 * b2   with b0 and b2 the same view of one store
    k = KProg(slots, (), 0, ((2, 1, (("store", 2, (0,), ("bin", "+", ("ld", 0, (0,)), ("ld", 1, (0,)))),
                                     ("store", 3, (0,), ("bin", "*", ("ld", 0, (0,)), ("ld", 2, (0,)))))),), False)
    x = np.arange(1.0, 9.0)
    y = np.arange(10.0, 18.0)
    ref_x, ref_out = x.copy(), np.zeros(8)
    interpret(k, {0: ref_x, 1: y, 2: ref_x, 3: ref_out}, (), {})
    m, ci = aliasing.plan(k, {0: 5, 1: 6, 2: 5, 3: 7}, {i: ((0,), (8,)) for i in range(4)})
    assert m == {0: 2} and not ci
    k2 = aliasing.rewrite(k, m)
    dev_x, dev_out = x.copy(), np.zeros(8)
    copies = {0: np.full(8, np.nan), 1: y.copy(), 2: dev_x, 3: dev_out}  # slot 0 unreferenced now
    interpret(k2, copies, (), {})
    assert np.array_equal(dev_x, ref_x) and np.array_equal(dev_out, ref_out)


def test_check_isolated_rejects_overlapping_claims():
    from fakedev import FakeLib
    from paper_2406_18109_b200.errors import ArenaViolation
    from paper_2406_18109_b200.executor import Executor
    from paper_2406_18109_b200.ir import ArgDesc, PartDesc, TaskDesc

    ex = Executor(shapes={0: (10,), 1: (10,)}, lib=FakeLib(0, 1))
    tile = PartDesc("tiling", (4,), (0,), ((1,),), (0,))
    wide = PartDesc("tiling", (5,), (0,), ((1,),), (0,))  # 5-wide tiles at stride... tile p -> [5p, 5p+5)
    shifted = PartDesc("tiling", (4,), (1,), ((1,),), (0,))
    ok = TaskDesc("COPY", (2,), (ArgDesc(0, tile, "R"), ArgDesc(1, tile, "W")))
    ex.check_isolated(ok, frozenset())
    cross_read = TaskDesc("COPY", (2,), (ArgDesc(1, shifted, "R"), ArgDesc(1, tile, "W")))
    with pytest.raises(ArenaViolation):
        ex.check_isolated(cross_read, frozenset())
    ex.check_isolated(TaskDesc("COPY", (2,), (ArgDesc(0, wide, "R"), ArgDesc(1, wide, "W"))), frozenset())


def test_graph_segments_replay_identical_launches(monkeypatch):
    """GpuSession's graph relaunch (Executor.drain) on the CPU stand-in: repeated launch segments are
    captured once and relaunched, and the heaps still equal the reference Session's."""
    import os
    import sys

    from conftest import reference_available

    ref_src = reference_available()
    if ref_src is None:
        pytest.skip("reference not importable")
    sys.dont_write_bytecode = True
    if ref_src not in sys.path:
        sys.path.insert(0, ref_src)
    from diffusekit.pipeline import Session, SessionConfig, run_events
    from diffusekit.trace import gen_benchmark
    from fakedev import FakeLib

    from paper_2406_18109_b200 import runtime
    from paper_2406_18109_b200.session import GpuSession

    monkeypatch.setattr(runtime, "load", lambda *a, **k: FakeLib(0, 1, device_model=True))
    monkeypatch.setenv("DK_HOST_INIT", "1")
    for name, kw in (("blackscholes_chain", dict(size=4096, nodes=2, iters=6)), ("jacobi", dict(size=16, nodes=4, iters=4))):
        ref = Session(SessionConfig())
        run_events(ref, gen_benchmark(name, **kw))
        gpu = GpuSession(SessionConfig(), device=0)
        run_events(gpu, gen_benchmark(name, **kw))
        for s in ref.live_store_ids():
            assert same_bits(gpu.heap.get(s), ref.heap.get(s)), (name, s)
        if name == "blackscholes_chain":
            gs = gpu.executor.graph_stats
            assert gs["captures"] >= 1 and gs["graph_launches"] >= 2, gs


@pytest.mark.parametrize("name", ["cg_csr_8x8_k2/fused", "cg_csr_6x12_k4/fused", "pcg_csr_8x8_k2/fused"])
def test_spmv_dot_epilogue_matches_reference(name):
    """DK_FUSE_SPMV_DOT: the SpMV emits p.q partials and the [DOT, DOT] window drops that reduction;
    heaps match the reference within rtol 1e-12 (the only change is the summation order of p.q)."""
    from conftest import load_golden
    from fakedev import FakeLib

    from paper_2406_18109_b200.executor import Executor
    from paper_2406_18109_b200.plan import PlanTrace

    case = {c["name"]: c for c in load_golden("bench_small.json.gz")}[name]
    tr = PlanTrace.from_json(case["trace"])
    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, lib=FakeLib(0, 1, device_model=True),
                  fuse_spmv_dot=True)
    for kind, ev in tr.events:
        if kind == "exec":
            ex.execute(ev.task, ev.kernel, ev.temp_positions)
        elif kind == "free":
            ex.free(ev)
    assert ex.spmv_dot_stats["consumed"] >= 3 and ex.spmv_dot_stats["consumed"] == ex.spmv_dot_stats["spmv"]
    for s, want in golden_arrays(case).items():
        got = ex.get(s)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(want)))))


def test_host_streamed_windows_in_gpusession(monkeypatch):
    """GpuSession streams a window whose inputs were assigned pinned host arrays: H2D, kernel and the
    D2H of stream_out stores in chunks (CPU stand-in); the results equal the reference Session's, and
    the e2e loop (assign x, y; flush; get out) returns out == x + y every iteration."""
    import sys

    from conftest import reference_available

    ref_src = reference_available()
    if ref_src is None:
        pytest.skip("reference not importable")
    if ref_src not in sys.path:
        sys.path.insert(0, ref_src)
    from diffusekit.pipeline import Session, SessionConfig, run_events, task_from_event
    from diffusekit.trace import CreatePartition, CreateStore, DropRef, Flush, TaskEvent, gen_blackscholes_chain, \
        partition_from_event
    from fakedev import FakeLib

    from paper_2406_18109_b200 import runtime
    from paper_2406_18109_b200.session import GpuSession

    monkeypatch.setattr(runtime, "load", lambda *a, **k: FakeLib(0, 1, device_model=True))
    monkeypatch.setenv("DK_HOST_INIT", "1")
    n = 1000
    ev = gen_blackscholes_chain(size=n, nodes=1, iters=8)
    its, cur = [], []
    for e in ev:
        cur.append(e)
        if isinstance(e, Flush):
            its.append(cur)
            cur = []
    s = GpuSession(SessionConfig())
    ref = Session(SessionConfig())

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

    hx, hy, ho = s.pinned((n,)), s.pinned((n,)), s.pinned((n,))
    s.stream_out(2, ho)
    rng = np.random.default_rng(5)
    for k, it in enumerate(its):
        feed(s, [e for e in it if isinstance(e, (CreateStore, CreatePartition))])
        feed(ref, [e for e in it if isinstance(e, (CreateStore, CreatePartition))])
        hx[:] = rng.integers(1, 10, n)
        hy[:] = rng.integers(1, 10, n)
        s.heap.arrays[0] = hx
        s.heap.arrays[1] = hy
        ref.heap.arrays[0] = hx.copy()
        ref.heap.arrays[1] = hy.copy()
        feed(s, [e for e in it if not isinstance(e, (CreateStore, CreatePartition))])
        feed(ref, [e for e in it if not isinstance(e, (CreateStore, CreatePartition))])
        got = s.heap.get(2, out=ho)
        assert got is ho and np.array_equal(ho, hx + hy), k
        assert np.array_equal(s.heap.get(2), ref.heap.get(2))
        assert np.array_equal(s.heap.get(0), hx)
    assert s.streamed_windows >= 5, s.streamed_windows
    s.close()


def test_builtin_input_overlapping_its_output_is_copied_in():
    """MATVEC whose vector operand and result are overlapping views of one store: numpy computes
    ``a0 @ a1`` before assigning (executor.py:93-94); the executor reads a copy."""
    from fakedev import FakeLib

    from paper_2406_18109_b200.executor import Executor
    from paper_2406_18109_b200.ir import ArgDesc, PartDesc, TaskDesc

    ex = Executor(shapes={0: (6, 6), 1: (8,)}, lib=FakeLib(0, 1, device_model=True))
    A = np.arange(36.0).reshape(6, 6) / 7.0
    v = np.arange(1.0, 9.0)
    ex.upload(0, A)
    ex.upload(1, v)
    whole = PartDesc("tiling", (6, 6), (0, 0), ((1,), (1,)), (0, 0))
    xin = PartDesc("tiling", (6,), (0,), ((1,),), (0,))
    yout = PartDesc("tiling", (6,), (2,), ((1,),), (0,))
    task = TaskDesc("MATVEC", (1,), (ArgDesc(0, whole, "R"), ArgDesc(1, xin, "R"), ArgDesc(1, yout, "W")))
    ex.execute(task, None)
    want = v.copy()
    want[2:8] = A @ v[0:6]
    assert np.allclose(ex.get(1), want, rtol=1e-15)
