"""CUDA-graph replay of a memo-hit iteration (dk_graph_*) gives the same heap.

The reference re-runs ``Session._replay`` (pipeline.py:278-286) and ``execute_task``
(executor.py:163-195) for every memo hit; here the last steady iteration of a golden plan is
captured from the library stream and launched as one graph instead.  The final heap must equal
the oracle's replay of the whole plan byte for byte (integer-valued heaps).
"""
import gzip
import json
import os

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(name):
    with gzip.open(os.path.join(REPO, "tests", "golden", "bench_small.json.gz"), "rt") as f:
        return next(c for c in json.load(f)["cases"] if c["name"] == name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["blackscholes_chain/fused", "stencil/fused"])
def test_graph_replay_of_last_iteration_matches_oracle(name):
    from paper_2406_18109_b200.executor import Executor, replay
    from paper_2406_18109_b200.plan import PlanTrace

    from oracle.interp import replay as oracle_replay

    trace = PlanTrace.from_json(_case(name)["trace"])
    its = trace.iterations()
    assert len(its) >= 3
    ex = Executor(shapes=trace.shapes, seed=trace.seed, init=trace.init, dtypes=trace.dtypes, device=0)
    try:
        for it in its[:-1]:
            replay(ex, it)
        ex.sync()
        n0 = ex.launch_count()
        g = ex.capture(lambda: replay(ex, its[-1]))
        assert ex.launch_count() == n0  # captured, not launched
        ex.graph_launch(g)
        ex.sync()
        assert ex.launch_count() > n0
        ex.graph_destroy(g)
        ref = oracle_replay(trace)
        for sid in trace.live:
            got, want = ex.get(sid), ref.get(sid)
            assert np.array_equal(got, want), f"store {sid} differs after graph replay"
    finally:
        ex.close()


@pytest.mark.gpu
def test_graph_capture_of_cooperative_multi_nest_window():
    """A multi-nest window (one cooperative launch with grid barriers) captured into a CUDA graph
    and relaunched leaves the same bytes as launching it directly a second time."""
    from paper_2406_18109_b200.executor import Executor, replay
    from paper_2406_18109_b200.plan import PlanTrace

    with gzip.open(os.path.join(REPO, "tests", "golden", "fuzz250.json.gz"), "rt") as f:
        cases = json.load(f)["cases"]
    done = 0
    for case in cases:
        trace = PlanTrace.from_json(case["trace"])
        ev = trace.events
        k = next((i for i, (kind, e) in enumerate(ev) if kind == "exec" and e.kernel is not None
                  and len(e.kernel.nests) > 1), None)
        if k is None:
            continue
        e = ev[k][1]
        outs = []
        for use_graph in (True, False):
            ex = Executor(shapes=trace.shapes, seed=trace.seed, init=trace.init, dtypes=trace.dtypes, device=0)
            try:
                replay(ex, ev[:k + 1])
                ex.sync()
                if use_graph:
                    g = ex.capture(lambda: ex.execute(e.task, e.kernel, e.temp_positions))
                    ex.graph_launch(g)
                    ex.sync()
                    ex.graph_destroy(g)
                else:
                    ex.execute(e.task, e.kernel, e.temp_positions)
                outs.append({a.store: ex.get(a.store) for j, a in enumerate(e.task.args)
                             if j not in e.temp_positions and a.store in ex.stores})
            finally:
                ex.close()
        for sid, want in outs[1].items():
            assert np.array_equal(outs[0][sid], want, equal_nan=True), (case["name"], sid)
        done += 1
        if done == 5:
            break
    assert done == 5
