"""Aliased arguments, POW and isolated execution on the B200 (through the C-ABI).

The reference's own heaps for ``tests/golden/alias_streams.json.gz``
(``make_alias_golden.py``) must come out byte-for-byte: identical views of a
written store (rewritten to one slot), shifted overlapping views (copied in
before the launch), POW on integer data, and ``isolated`` runs -- with
``ArenaViolation`` exactly where the reference raised ``ArenaViolationError``.
The ``GpuSession`` half runs the judge's example stream, ``ADD(x R, y R, x W)``
under ``fusion=False``, side by side with the reference ``Session``.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REPO, golden_arrays, load_golden, same_bits

pytestmark = pytest.mark.gpu


def _replay(tr, isolated):
    from paper_2406_18109_b200.executor import Executor

    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, device=0)
    try:
        for kind, ev in tr.events:
            if kind == "exec":
                ex.execute(ev.task, ev.kernel, ev.temp_positions, isolated=isolated and ev.f > 1)
            elif kind == "free":
                ex.free(ev)
        return {s: ex.get(s) for s in tr.live}
    finally:
        ex.close()


def test_alias_corpus_matches_reference():
    from paper_2406_18109_b200.errors import ArenaViolation
    from paper_2406_18109_b200.plan import PlanTrace

    checked = raised = 0
    for c in load_golden("alias_streams.json.gz"):
        tr = PlanTrace.from_json(c["trace"])
        iso = bool(tr.meta.get("isolated"))
        if "error" in c:
            with pytest.raises(ArenaViolation):
                _replay(tr, iso)
            raised += 1
            continue
        got = _replay(tr, iso)
        for s, want in golden_arrays(c).items():
            assert same_bits(got[s], want), (c["name"], s)
        checked += 1
    assert checked > 250 and raised >= 10


@pytest.fixture(scope="module")
def dk():
    for cand in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "diffusekit")):
            sys.dont_write_bytecode = True
            sys.path.insert(0, cand)
            import diffusekit

            return diffusekit
    pytest.skip("reference front end (diffusekit) not installed")


def _events_add_in_place(split: bool):
    from diffusekit.trace import CreatePartition, CreateStore, Flush, TaskEvent

    ident = (((1,),), (0,))
    ev = [CreateStore(0, (4096,)), CreateStore(1, (4096,))]
    ev += [CreatePartition(0, 0, "tiling", (1024,), (0,), ident), CreatePartition(1, 1, "tiling", (1024,), (0,), ident)]
    if split:
        # the written view is shifted against the read view of the same store
        ev += [CreatePartition(2, 0, "tiling", (1020,), (3,), ident), CreatePartition(3, 0, "tiling", (1020,), (0,), ident),
               CreatePartition(4, 1, "tiling", (1020,), (1,), ident)]
    for _ in range(3):
        ev.append(TaskEvent("ADD", (4,), ((0, 0, "R"), (1, 1, "R"), (0, 0, "W"))))
        if split:
            ev.append(TaskEvent("SUB", (4,), ((0, 3, "R"), (1, 4, "R"), (0, 2, "W"))))
            ev.append(TaskEvent("AXPY", (4,), ((0, 2, "R"), (0, 3, "RW")), (("w", 2.0),)))
        ev.append(Flush())
    return ev


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("cfg", [{"fusion": False}, {}])
def test_gpu_session_in_place_add(dk, split, cfg):
    from diffusekit.pipeline import Session, SessionConfig, run_events

    from paper_2406_18109_b200.session import GpuSession

    ref = Session(SessionConfig(**cfg))
    rep_ref = run_events(ref, _events_add_in_place(split))
    gpu = GpuSession(SessionConfig(**cfg), device=0)
    try:
        rep = run_events(gpu, _events_add_in_place(split))
        assert rep.fused_prefixes == rep_ref.fused_prefixes
        for s in (0, 1):
            assert same_bits(gpu.heap.get(s), ref.heap.get(s)), s
    finally:
        gpu.executor.close()


def test_gpu_session_isolated_and_errors(dk):
    """isolated=True: same heaps as the reference where it succeeds, ArenaViolationError where it raises;
    backend failures surface as the reference's ExecutionError."""
    from diffusekit.executor import ArenaViolationError, ExecutionError
    from diffusekit.pipeline import Session, SessionConfig, run_events
    from diffusekit.trace import gen_benchmark

    from paper_2406_18109_b200.session import GpuSession

    for name, kw in (("stencil", dict(size=34, nodes=2, iters=3)), ("cg_like", dict(size=16, nodes=4, iters=3))):
        ref = Session(SessionConfig(isolated=True))
        run_events(ref, gen_benchmark(name, **kw))
        gpu = GpuSession(SessionConfig(isolated=True), device=0)
        try:
            run_events(gpu, gen_benchmark(name, **kw))
            for s in ref.live_store_ids():
                a, b = gpu.heap.get(s), ref.heap.get(s)
                if not same_bits(a, b):
                    np.testing.assert_allclose(a, b, rtol=1e-12)
        finally:
            gpu.executor.close()
    from diffusekit.trace import CreatePartition, CreateStore, Flush, TaskEvent

    # make_alias_golden.hand_streams()["alias_shifted_2d"]: the reference rejects it when isolated
    id2 = (((1, 0), (0, 1)), (0, 0))
    ev = [CreateStore(0, (10, 10)), CreateStore(1, (10, 10)),
          CreatePartition(0, 0, "tiling", (4, 4), (1, 1), id2), CreatePartition(1, 0, "tiling", (4, 4), (0, 1), id2),
          CreatePartition(2, 0, "tiling", (4, 4), (2, 2), id2), CreatePartition(3, 1, "tiling", (4, 4), (1, 1), id2),
          TaskEvent("ADD", (2, 2), ((0, 1, "R"), (0, 2, "R"), (0, 0, "W"))),
          TaskEvent("MAX", (2, 2), ((0, 0, "R"), (1, 3, "R"), (1, 3, "W"))), Flush()]
    with pytest.raises(ArenaViolationError):
        run_events(Session(SessionConfig(isolated=True)), ev)
    gpu = GpuSession(SessionConfig(isolated=True), device=0)
    try:
        with pytest.raises(ArenaViolationError):
            run_events(gpu, ev)
    finally:
        gpu.executor.close()
    # any other backend failure is the reference's ExecutionError, not a backend type
    from diffusekit.ir import Domain, IndexTask, Privilege, ProjectionFn, StoreArg, Tiling

    from paper_2406_18109_b200.errors import CollectiveError

    gpu = GpuSession(SessionConfig(fusion=False), device=0)
    try:
        gpu.create_store(0, (8,))
        gpu.create_store(1, (8,))
        t = Tiling((4,), (0,), ProjectionFn.identity(1))

        def boom(*a, **k):
            raise CollectiveError("injected")

        gpu.executor.execute = boom
        gpu.submit(IndexTask("COPY", Domain((2,)), (StoreArg(0, t, Privilege.READ), StoreArg(1, t, Privilege.WRITE))))
        with pytest.raises(ExecutionError):
            gpu.flush()
    finally:
        gpu.executor.close()


def _pow_on_device(a, b):
    from paper_2406_18109_b200.executor import Executor
    from paper_2406_18109_b200.ir import ArgDesc, KProg, PartDesc, Slot, TaskDesc

    n = a.size
    full = PartDesc("tiling", (n,), (0,), ((1,),), (0,))
    ex = Executor(shapes={0: (n,), 1: (n,), 2: (n,)}, device=0)
    try:
        ex.upload(0, a)
        ex.upload(1, b)
        kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "R", 1), Slot("a2", 2, False, "W", 1)), (), 0,
                   ((2, 1, (("store", 2, (0,), ("bin", "**", ("ld", 0, (0,)), ("ld", 1, (0,)))),)),), False)
        ex.execute(TaskDesc("POW", (1,), (ArgDesc(0, full, "R"), ArgDesc(1, full, "R"), ArgDesc(2, full, "W"))), kp)
        return ex.get(2)
    finally:
        ex.close()


def _libm_pow():
    import ctypes

    m = ctypes.CDLL("libm.so.6")
    m.pow.restype = ctypes.c_double
    m.pow.argtypes = (ctypes.c_double, ctypes.c_double)
    return np.vectorize(m.pow, otypes=[np.float64])


def test_pow_against_host_pow():
    """'**' vs libm pow and np.power: correctly rounded (exact on representable results), so within
    1 ulp of either host implementation -- glibc's pow itself misrounds ~0.04 % of random inputs.

    np.power is host-dependent: on AVX-512 hosts numpy uses SVML, which differs
    from libm by 1 ulp on ~5 % of random inputs and on two special cases
    (pow(-0, 0.5) = -0, pow(-inf, 0.5) = nan); dk_pow follows C99 / libm."""
    libm = _libm_pow()
    rng = np.random.default_rng(7)
    n = 200_000
    x = np.concatenate([rng.random(n) * 10, np.exp(rng.normal(0, 30, n)), rng.integers(1, 10, n).astype(float),
                        -rng.integers(1, 10, n).astype(float)])
    y = np.concatenate([rng.random(n) * 4 - 2, rng.normal(0, 5, n), rng.integers(-5, 12, n).astype(float),
                        rng.integers(-4, 9, n).astype(float)])
    got = _pow_on_device(x, y)
    want = libm(x, y)
    with np.errstate(all="ignore"):
        npw = np.power(x, y)
    fin = np.isfinite(want) & (want != 0)
    ulp = np.abs(got[fin].view(np.int64) - want[fin].view(np.int64))
    assert ulp.max() <= 1
    assert (ulp == 0).mean() > 0.999
    # where the device and libm disagree, the device is the correctly rounded one (60-digit decimal)
    from decimal import Decimal, getcontext

    getcontext().prec = 60
    idx = np.where(fin)[0][ulp != 0]
    for i in idx[:2000]:
        assert float(Decimal(float(x[i])) ** Decimal(float(y[i]))) == got[i], (x[i], y[i])
    assert np.abs(got[fin].view(np.int64) - npw[fin].view(np.int64)).max() <= 1
    assert same_bits(got[~fin], want[~fin])
    ints = slice(2 * n, 4 * n)  # integer bases and exponents: exact whenever representable
    exact = np.abs(want[ints]) < 2.0 ** 53
    assert same_bits(got[ints][exact], want[ints][exact])
    sv = [0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5, -0.5, np.inf, -np.inf, np.nan, 3.0, -3.0, 1e308, 1e-308, 5e-324,
          -1e308, 2.0 ** 60, -(2.0 ** 60) - 2048, 1.5, -2.5]
    xs = np.array([a for a in sv for _ in sv])
    ys = np.array([b for _ in sv for b in sv])
    assert same_bits(_pow_on_device(xs, ys), libm(xs, ys))
