"""Host-streamed execution (streaming.HostStreamer) gives the executor's results."""

import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_streamed_blackscholes_window_matches_oracle():
    from oracle.interp import OracleHeap, execute_step
    from paper_2406_18109_b200.executor import Executor
    from paper_2406_18109_b200.plan import PlanTrace
    from paper_2406_18109_b200.streaming import HostStreamer, pinned

    with gzip.open(os.path.join(GOLDEN, "plans_medium.json.gz"), "rt") as f:
        traces = {t["meta"]["name"]: PlanTrace.from_json(t) for t in json.load(f)["traces"]}
    for name in ("bs_1e5_k1/fused", "bs_1e5_k2/fused"):
        tr = traces[name]
        big = [e for e in tr.execs() if e.f == 67][-1]
        x, y = big.task.args[0].store, big.task.args[1].store
        out = [a.store for a in big.task.args if a.priv == "W" and a.store in tr.live][-1]
        ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, device=0)
        try:
            hx, _ = pinned(ex, tr.shapes[x])
            hy, _ = pinned(ex, tr.shapes[y])
            ho, _ = pinned(ex, tr.shapes[out])
            rng = np.random.default_rng(7)
            hx[:] = rng.random(hx.shape)
            hy[:] = rng.integers(-5, 5, hy.shape)
            st = HostStreamer(ex, chunks=5)
            for _ in range(2):
                st.run(big.task, big.kernel, big.temp_positions, {x: hx, y: hy}, {out: ho})
            ex.sync()
            heap = OracleHeap(tr.shapes, tr.seed, tr.init)
            heap.arrays[x] = hx.copy()
            heap.arrays[y] = hy.copy()
            execute_step(big, heap)
            assert np.array_equal(ho, heap.get(out)), name
            # the device copy is coherent with the host result
            assert np.array_equal(ex.get(out), ho)
        finally:
            ex.close()
