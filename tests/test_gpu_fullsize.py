"""Parity at the BASELINE sizes (north star: fp64 within rtol 1e-12, residual histories within 1e-10).

The recorded full-size plans the bench times (``paper_2406_18109_b200/workloads``:
the 32768^2 stencil with residual, CG and Jacobi-PCG on the 67M-row Poisson
matrix) run through the executor on the B200 and through the CPU oracle on
the same initial contents (``oracle.interp`` in its chunked, threaded mode
with the C ``SPMV_CSR``; pinned by ``tests/test_oracle_golden.py``).

* Stencil: no value depends on a reduction, so ``grid`` and ``work`` must be
  **bit-identical** after every iteration run; each ``res`` (the residual
  history, one rank-0 store per iteration) within rtol 1e-12 -- the only
  difference is the summation order of the reduction.
* CG / PCG, two ways:
  - *lockstep*: after every window the oracle's reduction targets (pq,
    rs_old, rs_new / rz_*) are checked against the device's at rtol 1e-12
    and then replaced by the device's values, so both sides feed identical
    scalars into the next window; every vector (x, r, p, q, z, resid) must
    then be **bit-identical** -- the SpMV and every vector window round
    exactly like numpy;
  - *free-running*: the oracle runs on its own; the residual histories
    (rs_new / rz_new per iteration) agree within 1e-10 relative and the
    vectors within rtol 1e-10 (atol 1e-10 x max|v|).
"""

import gzip
import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN, REPO, same_bits

pytestmark = pytest.mark.gpu

ITERS = 12  # >= 10 steady iterations after the ramp (the plans hold 24)
WORKERS = max(1, min(16, os.cpu_count() or 1))


def _trace(name):
    from paper_2406_18109_b200.plan import PlanTrace

    return PlanTrace.load(os.path.join(REPO, "paper_2406_18109_b200", "workloads", name + ".json.gz"))


def _large(name):
    from paper_2406_18109_b200.plan import PlanTrace

    with gzip.open(os.path.join(GOLDEN, "plans_large.json.gz"), "rt") as f:
        return {t["meta"]["name"]: PlanTrace.from_json(t) for t in json.load(f)["traces"]}[name]


@pytest.fixture(autouse=True)
def _shared_poisson(monkeypatch):
    """The executor and the oracle both build the Poisson CSR tiles on the host: build each once."""
    import functools
    import importlib

    executor = importlib.import_module("paper_2406_18109_b200.executor")
    initheap = importlib.import_module("paper_2406_18109_b200.initheap")

    cached = functools.lru_cache(maxsize=2)(initheap.poisson_tile)
    monkeypatch.setattr(initheap, "poisson_tile", cached)
    monkeypatch.setattr(executor, "poisson_tile", cached)
    yield
    cached.cache_clear()


def _red_targets(step, shapes):
    return sorted({a.store for a in step.task.args if a.reduces and shapes[a.store] == ()})


def _run(tr, iters, lockstep, fuse_spmv_dot=False):
    """Device replay of the first ``iters`` iterations; with ``lockstep`` the oracle runs window by
    window beside it and takes the device's reduction results.  Returns (executor, oracle heap, rank-0 log)."""
    from oracle.interp import OracleHeap, execute_step, parallel
    from paper_2406_18109_b200.executor import Executor

    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, device=0,
                  fuse_spmv_dot=fuse_spmv_dot)
    oh = OracleHeap(tr.shapes, tr.seed, tr.init) if lockstep else None
    worst = 0.0
    with parallel(WORKERS):
        for it in tr.iterations()[:iters]:
            for kind, ev in it:
                if kind == "exec":
                    ex.execute(ev.task, ev.kernel, ev.temp_positions)
                    if lockstep:
                        execute_step(ev, oh)
                        for sid in _red_targets(ev, tr.shapes):
                            g = float(ex.get(sid)[()])
                            w = float(oh.get(sid)[()])
                            worst = max(worst, abs(g - w) / max(abs(w), 1e-300))
                            oh.arrays[sid][()] = g
                elif kind == "free":
                    ex.free(ev)
                    if lockstep:
                        oh.free(ev)
    ex.sync()
    return ex, oh, worst


def _oracle(tr, iters):
    from oracle.interp import OracleHeap, replay

    oh = OracleHeap(tr.shapes, tr.seed, tr.init)
    for it in tr.iterations()[:iters]:
        replay(tr, it, oh, workers=WORKERS)
    return oh


def _alive(ex, oh):
    return sorted(s for s in oh.arrays if s in ex.stores)


def _check_stencil(tr, iters):
    t0 = time.time()
    ex, _, _ = _run(tr, iters, lockstep=False)
    t1 = time.time()
    try:
        oh = _oracle(tr, iters)
        t2 = time.time()
        n_big = n_res = 0
        for s in _alive(ex, oh):
            g, w = ex.get(s), oh.get(s)
            if tr.shapes[s] == ():
                np.testing.assert_allclose(g, w, rtol=1e-12, err_msg=f"res store {s}")
                n_res += 1
            else:
                assert same_bits(g, w), f"store {s} {tr.shapes[s]} not bit-identical"
                n_big += 1
            del g
        assert n_big >= 2 and n_res >= iters - 1
        print(f"{tr.meta.get('name')}: device {t1 - t0:.1f}s oracle {t2 - t1:.1f}s check {time.time() - t2:.1f}s")
    finally:
        ex.close()


def test_stencil_32768_fused_sweep_residual():
    """BASELINE configs[2] on one GPU: 32768^2 interior, 12 iterations of [ADD x4, MULT, SUB, DOT][COPY]."""
    tr = _trace("stencil_fused_n1")
    assert tr.shapes[0] == (32770, 32770)
    _check_stencil(tr, ITERS)


@pytest.mark.parametrize("mode,iters", [("fused", ITERS), ("unfused", 6)])
def test_stencil_four_bands_one_gpu(mode, iters):
    """Four 8192^2 row bands as four launch points on one GPU (the partitioned plan shape)."""
    _check_stencil(_large(f"stencil_8192_k4/{mode}"), iters)


@pytest.mark.parametrize("name,iters", [("cg_fused_n1", ITERS), ("pcg_fused_n1", ITERS), ("cg_unfused_n1", 6)])
def test_cg_lockstep_bit_identical(name, iters):
    """BASELINE configs[3]/[4] (67M rows): with identical scalars every vector is bit-identical."""
    tr = _trace(name)
    assert tr.shapes[3] == (8192 * 8192,)
    t0 = time.time()
    ex, oh, worst = _run(tr, iters, lockstep=True)
    try:
        assert worst <= 1e-12, f"reduction results differ by {worst:.3g} relative"
        vecs = [s for s in _alive(ex, oh) if tr.shapes[s] != () and tr.dtypes.get(s, "f64") == "f64"
                and not tr.init.get(s, {}).get("kind", "").startswith("csr")]
        assert len(vecs) >= 5
        for s in vecs:
            assert same_bits(ex.get(s), oh.get(s)), f"vector store {s} not bit-identical"
        print(f"{name}: lockstep {time.time() - t0:.1f}s, reductions within {worst:.2e}")
    finally:
        ex.close()


@pytest.mark.parametrize("name,fuse", [("cg_fused_n1", False), ("pcg_fused_n1", False), ("cg_fused_n1", True)])
def test_cg_free_running_residual_history(name, fuse):
    """Device and oracle each on their own: rs_new / rz_new histories within 1e-10 relative
    (``fuse``: with the opt-in SpMV + partial-dot epilogue, DK_FUSE_SPMV_DOT)."""
    tr = _trace(name)
    t0 = time.time()
    ex, _, _ = _run(tr, ITERS, lockstep=False, fuse_spmv_dot=fuse)
    if fuse:
        assert ex.spmv_dot_stats["consumed"] >= ITERS - 1
    try:
        oh = _oracle(tr, ITERS)
        alive = _alive(ex, oh)
        hist = [s for s in alive if tr.shapes[s] == () and s in tr.live]
        assert len(hist) >= ITERS - 1
        g = np.array([float(ex.get(s)[()]) for s in hist])
        w = np.array([float(oh.get(s)[()]) for s in hist])
        assert np.all(w > 0)  # (the 2-norm of the CG residual is not monotone: it grows here at first)
        np.testing.assert_allclose(g, w, rtol=1e-10)
        for s in alive:
            if tr.shapes[s] != () and not tr.init.get(s, {}).get("kind", "").startswith("csr"):
                a, b = ex.get(s), oh.get(s)
                np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10 * float(np.max(np.abs(b))),
                                           err_msg=f"store {s}")
        print(f"{name}: free-running {time.time() - t0:.1f}s, history {g[0]:.6e} -> {g[-1]:.6e}")
    finally:
        ex.close()
