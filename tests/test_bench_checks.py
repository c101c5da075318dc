"""bench.py's post-run result checks, exercised on CPU with the device stand-in (fakedev).

The checks run one more iteration of each full-size workload after the timed
region and verify it by the workload's identities (stencil update and residual,
CG recurrence vs true residual, ...).  Here they run on the bounded CPU plans;
a corrupted device value must turn them into FAILED.
"""

import importlib.util
import os

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _host_init(monkeypatch):
    monkeypatch.setenv("DK_HOST_INIT", "1")  # the stand-in has no device PCG64


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_checks_mod", os.path.join(REPO, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _setup(bench, name, n_its):
    from fakedev import FakeLib
    from paper_2406_18109_b200.executor import Executor, replay

    tr = bench.load_trace(name)
    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, lib=FakeLib(0, 1))
    its, steady = bench.iteration_split(tr)
    for i in range(n_its):
        replay(ex, its[i])
    return ex, tr, its


@pytest.mark.parametrize("wl,name", [("stencil", "stencil_fused_cpu"), ("cg", "cg_fused_cpu"),
                                     ("pcg", "pcg_fused_cpu"), ("stencil", "stencil_unfused_cpu"),
                                     ("cg", "cg_unfused_cpu"), ("pcg", "pcg_unfused_cpu"),
                                     ("bs", "bs_fused_c1"), ("bs", "bs_unfused_c1")])
def test_result_check_passes(bench, wl, name):
    ex, tr, its = _setup(bench, name, 4)
    out = bench.result_check(ex, tr, wl, its, 4, None, 1)
    assert out["status"] == "ok", out


def test_result_check_catches_corruption(bench):
    import numpy as np

    ex, tr, its = _setup(bench, "cg_fused_cpu", 4)
    # corrupt one entry of x: the recurrence residual no longer matches b - A x
    x = ex.get(3)
    x[12345] += 1e-3
    ex.upload(3, x)
    out = bench.result_check(ex, tr, "cg", its, 4, None, 1)
    assert out["status"] == "FAILED" and out["true_residual_gap"] > 1e-9
    ex, tr, its = _setup(bench, "stencil_fused_cpu", 3)
    lib = ex.lib
    orig = lib.dk_launch

    def bad_launch(h, views, nviews, scalars, nscal, totals):
        rc = orig(h, views, nviews, scalars, nscal, totals)
        if nviews >= 6:  # the fused sweep: perturb one element of work afterwards
            w = lib._store_array(1)
            w[7, 9] = np.nextafter(w[7, 9], np.inf)
        return rc

    lib.dk_launch = bad_launch
    out = bench.result_check(ex, tr, "stencil", its, 3, None, 1)
    assert out["status"] == "FAILED" and not out["work_bit_identical"]
