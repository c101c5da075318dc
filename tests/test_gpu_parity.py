"""GPU parity: recorded reference plans replayed through the B200 executor.

* golden cases: the final heap must equal the reference's own bytes -- exactly
  when the reference heap is integer-valued (all arithmetic exact), else
  within rtol 1e-12 (north star; reduction order differs from np.sum);
* medium plans: compared with the CPU oracle on the same inputs;
* edge cases: empty/clamped sub-stores, broadcasting, privilege and bounds
  errors, NaN/-0.0 semantics.
"""

import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_arrays, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Executor():
    from paper_2406_18109_b200.executor import Executor as E

    return E


def _run(Executor, trace, world=1):
    from paper_2406_18109_b200.executor import replay

    ex = Executor(shapes=trace.shapes, seed=trace.seed, init=trace.init, dtypes=trace.dtypes, device=0)
    try:
        replay(ex, trace.events)
        return {s: ex.get(s) for s in trace.live}, ex
    finally:
        ex.close()


def _compare(name, got, want, exact, trace=None):
    """``exact``: every store bit-identical.  Otherwise stores a reduction result can reach
    (``_reduction_reach``) within rtol 1e-12 -- a reduction's summation order differs from
    np.sum -- and every other store still bit-identical (no FMA, IEEE-exact elementwise ops)."""
    reach = _reduction_reach(trace) if (trace is not None and not exact) else None
    for s, w in want.items():
        g = got[s]
        if exact or (reach is not None and s not in reach):
            assert same_bits(g, w), f"{name}: store {s} not bit-identical"
        else:
            np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(w)))),
                                       err_msg=f"{name}: store {s}")


def _reduction_reach(trace):
    """Stores whose final contents can depend on a reduction result: the reduction targets and,
    transitively, every store written by a launch that reads a reached store."""
    reach = set()
    changed = True
    execs = trace.execs()
    while changed:
        changed = False
        for e in execs:
            args = [a for j, a in enumerate(e.task.args) if j not in e.temp_positions]
            new = {a.store for a in args if a.reduces}
            # a launch (a fused window included: its demoted temporaries stay inside it) that reads
            # a reached store can pass it on to everything it writes
            if any(a.reads and a.store in reach for a in args):
                new |= {a.store for a in args if a.writes or a.reduces}
            if not new <= reach:
                reach |= new
                changed = True
    return reach


def _integer_valued(arrs):
    return all(np.all(np.isfinite(a)) and np.all(a == np.round(a)) for a in arrs.values())


def test_golden_bench_cases(Executor, bench_cases):
    from paper_2406_18109_b200.plan import PlanTrace

    exact_cases = 0
    for case in bench_cases:
        trace = PlanTrace.from_json(case["trace"])
        got, _ = _run(Executor, trace)
        want = golden_arrays(case)
        exact = _integer_valued(want)
        exact_cases += exact
        _compare(case["name"], got, want, exact, trace)
    assert exact_cases >= 5


def test_multi_nest_windows_run_as_one_launch(Executor, fuzz_cases, monkeypatch):
    """Fuzz windows with several nests run as ONE cooperative kernel per point (grid barriers
    between the nests): the reference's bytes either way, and DK_JIT_SPLIT_NESTS=1 (one launch
    per nest) costs exactly the extra nests' launches."""
    from ctypes import byref, c_int64

    from paper_2406_18109_b200.plan import PlanTrace

    def launches(ex):
        c = c_int64()
        ex.lib.dk_launch_count(byref(c))
        return c.value

    def run(trace):
        from paper_2406_18109_b200.executor import replay

        ex = Executor(shapes=trace.shapes, seed=trace.seed, init=trace.init, dtypes=trace.dtypes, device=0)
        try:
            l0 = launches(ex)
            replay(ex, trace.events)
            ex.sync()
            n = launches(ex) - l0
            return {s: ex.get(s) for s in trace.live}, n
        finally:
            ex.close()

    saved = expect = ncases = 0
    for case in fuzz_cases:
        trace = PlanTrace.from_json(case["trace"])
        extra = 0
        for e in trace.execs():
            if e.kernel is not None and len(e.kernel.nests) > 1:
                pts = 1
                for d in e.task.launch:
                    pts *= d
                extra += (len(e.kernel.nests) - 1) * pts
        if not extra:
            continue
        want = golden_arrays(case)
        got, lm = run(trace)
        _compare(case["name"], got, want, _integer_valued(want), trace)
        monkeypatch.setenv("DK_JIT_SPLIT_NESTS", "1")
        got, ls = run(trace)
        monkeypatch.delenv("DK_JIT_SPLIT_NESTS")
        _compare(case["name"] + "/split", got, want, _integer_valued(want), trace)
        assert ls >= lm
        saved += ls - lm
        expect += extra
        ncases += 1
        if ncases == 30:
            break
    assert ncases >= 10 and saved == expect, (ncases, saved, expect)


def test_golden_fuzz_corpus(Executor, fuzz_cases):
    from paper_2406_18109_b200.plan import PlanTrace

    for case in fuzz_cases:
        trace = PlanTrace.from_json(case["trace"])
        got, _ = _run(Executor, trace)
        want = golden_arrays(case)
        _compare(case["name"], got, want, _integer_valued(want), trace)


def test_medium_plans_match_oracle(Executor):
    from oracle.interp import replay as oracle_replay
    from paper_2406_18109_b200.plan import PlanTrace

    with gzip.open(os.path.join(GOLDEN, "plans_medium.json.gz"), "rt") as f:
        traces = [PlanTrace.from_json(t) for t in json.load(f)["traces"]]
    for tr in traces:
        got, _ = _run(Executor, tr)
        ref = oracle_replay(tr)
        want = {s: ref.get(s) for s in tr.live}
        name = tr.meta.get("name", "?")
        # integer-valued heaps bit-exact throughout; otherwise only what a reduction result
        # reaches is compared at rtol (the stencil's res histories; CG's vectors via pq / rs)
        _compare(name, got, want, _integer_valued(want), tr)


_VARIANT_SCRIPT = r"""
import gzip, json, os, sys
sys.path.insert(0, os.path.join(os.environ["DK_REPO"], "tests"))
sys.path.insert(0, os.environ["DK_REPO"])
import test_gpu_parity as T
from paper_2406_18109_b200.executor import Executor
from paper_2406_18109_b200.plan import PlanTrace
from oracle.interp import replay as oracle_replay
with gzip.open(os.path.join(T.GOLDEN, "plans_medium.json.gz"), "rt") as f:
    traces = [PlanTrace.from_json(t) for t in json.load(f)["traces"]]
n = 0
for tr in traces:
    name = tr.meta["name"]
    if not name.startswith(tuple(os.environ.get("DK_VARIANT_PLANS", "stencil").split(","))):
        continue
    got, _ = T._run(Executor, tr)
    ref = oracle_replay(tr)
    T._compare(name, got, {s: ref.get(s) for s in tr.live}, False, tr)
    n += 1
print("checked", n)
"""


@pytest.mark.parametrize("variant", ["DK_JIT_NO_K3", "DK_JIT_H", "DK_JIT_NO_SHIFT", "DK_JIT_PERSIST", "DK_K3_CYCLIC", "DK_K3_REUSE",
                                     "DK_K3_TR=12", "DK_K3_TR=16", "DK_K3S=1", "DK_K3_NOWS=1"])
def test_stencil_codegen_variants_match_oracle(variant, tmp_path):
    """The stencil plans with the TMA-staged window (K3) off, the shuffled
    odd-offset pairs ('H') on, the shifted pair grid off, or persistent
    grid-stride CTAs instead of one CTA per chunk: every code path of the pair loop is checked against the oracle (a fresh process per variant:
    modules are cached per process)."""
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DK_REPO=repo, DK_JIT_CACHE=str(tmp_path))
    key, _, val = variant.partition("=")
    env[key] = val or "1"
    out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "checked 12" in out.stdout


@pytest.mark.parametrize("variant", ["DK_SPMV_PERSIST"])
def test_spmv_variants_match_oracle(variant, tmp_path):
    """CG / PCG plans with the persistent-grid SPMV_CSR kernel."""
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DK_REPO=repo, DK_JIT_CACHE=str(tmp_path), DK_VARIANT_PLANS="cg,pcg")
    env[variant] = "1"
    out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "checked 0" not in out.stdout


def test_cg_residual_history(Executor):
    """CG residual history (rs_new per iteration) within 1e-10 relative of the oracle."""
    from oracle.interp import replay as oracle_replay
    from paper_2406_18109_b200.plan import PlanTrace

    with gzip.open(os.path.join(GOLDEN, "plans_medium.json.gz"), "rt") as f:
        traces = {t["meta"]["name"]: PlanTrace.from_json(t) for t in json.load(f)["traces"]}
    for name in ("cg_64x64_k2/fused", "pcg_64x64_k2/fused", "cg_64x128_k4/unfused"):
        tr = traces[name]
        got, _ = _run(Executor, tr)
        ref = oracle_replay(tr)
        hist = [s for s in tr.live if tr.shapes[s] == ()]
        assert len(hist) >= 6
        g = np.array([got[s] for s in hist], dtype=np.float64)
        w = np.array([ref.get(s) for s in hist], dtype=np.float64)
        assert np.all(w[1:] < w[0] * 10)
        np.testing.assert_allclose(g, w, rtol=1e-10)


def test_kernel_errors_map_to_reference_exceptions(Executor):
    from paper_2406_18109_b200.errors import PrivilegeError, UnknownTaskKind
    from paper_2406_18109_b200.ir import ArgDesc, KProg, PartDesc, Slot, TaskDesc

    tile = PartDesc("tiling", (4,), (0,), ((1,),), (0,))
    ex = Executor(shapes={0: (8,), 1: (8,)}, device=0)
    try:
        # store into a read-only parameter
        kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "R", 1)), (), 0,
                   ((1, 1, (("store", 1, (0,), ("ld", 0, (0,))),)),), False)
        task = TaskDesc("COPY", (2,), (ArgDesc(0, tile, "R"), ArgDesc(1, tile, "R")))
        with pytest.raises(PrivilegeError):
            ex.execute(task, kp)
        with pytest.raises(UnknownTaskKind):
            ex.execute(TaskDesc("MYSTERY", (2,), (ArgDesc(0, tile, "W"),)), None)
    finally:
        ex.close()


def test_nan_signed_zero_min_max_semantics(Executor):
    """np.minimum/np.maximum/np.negative bit semantics, including NaN and -0.0."""
    from paper_2406_18109_b200.ir import ArgDesc, KProg, PartDesc, Slot, TaskDesc

    a = np.array([0.0, -0.0, np.nan, 1.0, 2.0, -3.0, np.inf, -np.inf])
    b = np.array([-0.0, 0.0, 1.0, np.nan, 2.0, 5.0, np.nan, 1.0])
    full = PartDesc("tiling", (8,), (0,), ((1,),), (0,))
    for op, ref in (("min", np.minimum), ("max", np.maximum), ("/", np.true_divide), ("lt", np.less), ("eq", np.equal)):
        ex = Executor(shapes={0: (8,), 1: (8,), 2: (8,)}, device=0)
        try:
            ex.upload(0, a)
            ex.upload(1, b)
            kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "R", 1), Slot("a2", 2, False, "W", 1)), (),
                       0, ((2, 1, (("store", 2, (0,), ("bin", op, ("ld", 0, (0,)), ("ld", 1, (0,)))),)),), False)
            ex.execute(TaskDesc("X", (1,), (ArgDesc(0, full, "R"), ArgDesc(1, full, "R"), ArgDesc(2, full, "W"))), kp)
            got = ex.get(2)
            with np.errstate(all="ignore"):
                want = ref(a, b).astype(np.float64)
            assert np.array_equal(np.signbit(got[~np.isnan(want)]), np.signbit(want[~np.isnan(want)])), op
            assert same_bits(got, want), op
        finally:
            ex.close()
    ex = Executor(shapes={0: (8,), 1: (8,)}, device=0)
    try:
        ex.upload(0, a)
        kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "W", 1)), (), 0,
                   ((1, 1, (("store", 1, (0,), ("neg", ("ld", 0, (0,)))),)),), False)
        ex.execute(TaskDesc("NEG", (1,), (ArgDesc(0, full, "R"), ArgDesc(1, full, "W"))), kp)
        got = ex.get(1)
        assert np.array_equal(np.signbit(got), np.signbit(np.negative(a)))
    finally:
        ex.close()


def test_device_pcg64_init_matches_numpy(Executor):
    """dk_pcg64_fill reproduces default_rng([seed, sid]).integers(1, 10) / .random() bit for bit."""
    from paper_2406_18109_b200.initheap import host_contents

    cases = [
        ((300_001,), None, [((0,), (300_001,))]),
        ((700, 513), None, [((0, 0), (700, 513)), ((3, 1), (650, 512)), ((0, 0), (1, 513)), ((699, 0), (700, 513))]),
        ((1000, 300), None, [((0, 0), (1000, 1)), ((0, 299), (1000, 300)), ((17, 5), (18, 250))]),
        ((250_000,), {"kind": "uniform", "seed": 0, "key": 1000}, [((5,), (249_990,))]),
        ((250_000,), {"kind": "uniform", "seed": 0, "key": 1000, "scale": 0.25}, [((0,), (250_000,))]),
    ]
    for seed in (0, 3):
        for sid, (shape, spec, rects) in enumerate(cases):
            ex = Executor(shapes={sid: shape}, seed=seed, init={sid: spec} if spec else {}, device=0)
            try:
                r = ex.rec(sid)
                ex._materialize_init(r, rects)
                for o in range(ex.world):
                    r.valid[o] = list(rects)
                want = host_contents(spec, seed, sid, shape)
                got = np.full(shape, np.nan)
                for rect in rects:
                    ex.download_local(sid, got, rect)
                    sl = tuple(slice(l, h) for l, h in zip(*rect))
                    assert np.array_equal(got[sl], want[sl]), (seed, sid, rect)
            finally:
                ex.close()


def test_device_pcg64_rejection_path(Executor):
    """A stream with an early Lemire rejection: the element->draw shift must match numpy."""
    import ctypes

    from paper_2406_18109_b200.runtime import check

    ex = Executor(shapes={}, device=0)
    try:
        found = None
        for sid in range(4000):
            s = np.random.default_rng([0, sid]).bit_generator.state["state"]
            m64 = (1 << 64) - 1
            st = (ctypes.c_uint64 * 2)(s["state"] >> 64, s["state"] & m64)
            inc = (ctypes.c_uint64 * 2)(s["inc"] >> 64, s["inc"] & m64)
            out = (ctypes.c_int64 * 64)()
            n = ctypes.c_int64()
            check(ex.lib.dk_pcg64_rejects(st, inc, 3_000_000, out, 64, ctypes.byref(n)))
            if n.value:
                found = (sid, out[0])
                break
        assert found is not None, "no early rejection found"
        sid, q = found
        n = int(q) + 5000
        ex.shapes[sid] = (n,)
        r = ex.rec(sid)
        ex._materialize_init(r, [((0,), (n,))])
        r.valid[0] = [((0,), (n,))]
        got = np.empty(n)
        ex.download_local(sid, got, ((0,), (n,)))
        want = np.random.default_rng([0, sid]).integers(1, 10, size=n).astype(np.float64)
        assert np.array_equal(got, want)
        assert r.pcg is not None and len(r.pcg[1]) >= 1
    finally:
        ex.close()


def test_spmv_dot_epilogue_golden(Executor, bench_cases):
    """DK_FUSE_SPMV_DOT on the reference's CG / PCG golden cases: the SpMV kernel's partial-dot
    epilogue replaces the window's p.q reduction; heaps within rtol 1e-12 of the reference."""
    from paper_2406_18109_b200.executor import replay
    from paper_2406_18109_b200.plan import PlanTrace

    n = 0
    for case in bench_cases:
        if not case["name"].startswith(("cg_csr", "pcg_csr")) or not case["name"].endswith("/fused"):
            continue
        trace = PlanTrace.from_json(case["trace"])
        ex = Executor(shapes=trace.shapes, seed=trace.seed, init=trace.init, dtypes=trace.dtypes, device=0,
                      fuse_spmv_dot=True)
        try:
            replay(ex, trace.events)
            assert ex.spmv_dot_stats["consumed"] >= 3
            _compare(case["name"], {s: ex.get(s) for s in trace.live}, golden_arrays(case), False)
            n += 1
        finally:
            ex.close()
    assert n >= 3


def test_norm_builtin_grid_wide(Executor):
    """NORM (acc += sum(x*x), executor.py:97-98) on 3M elements: the grid-wide deterministic kernel
    (per-CTA partials folded in order) against numpy, accumulating onto the target's contents, and
    run-to-run bit-identical."""
    from paper_2406_18109_b200.ir import NONE_PART, ArgDesc, PartDesc, TaskDesc

    n = 3_000_001
    x = np.random.default_rng(11).random(n) - 0.25
    full = PartDesc("tiling", (n,), (0,), ((1,),), (0,))
    res = []
    for _ in range(2):
        ex = Executor(shapes={0: (n,), 1: ()}, device=0)
        try:
            ex.upload(0, x)
            ex.upload(1, np.array(2.5))
            task = TaskDesc("NORM", (1,), (ArgDesc(0, full, "R"), ArgDesc(1, NONE_PART, "Rd")))
            ex.execute(task, None)
            ex.execute(task, None)
            res.append(float(ex.get(1)[()]))
        finally:
            ex.close()
    want = 2.5 + 2 * float(np.sum(x * x))
    assert abs(res[0] - want) <= 1e-12 * want
    assert res[0] == res[1]
