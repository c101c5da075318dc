"""Workload for compute-sanitizer (racecheck / synccheck / memcheck) on one GPU.

    compute-sanitizer --tool racecheck python tools/gpu/sanitize_run.py

Replays medium plans that exercise the kernels with shared-memory protocols --
the K3 TMA/mbarrier stencil ring (stencil plans), the bulk-copy SPMV_CSR ring
(cg_64x64_k1: 4096 rows, one chunk ring per CTA), the reduction epilogue
(last-CTA fold) -- and the Black-Scholes window, and checks each against the
oracle.  Prints one line per plan; exit 1 on a mismatch.
"""

import gzip
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402

from oracle.interp import replay as oracle_replay  # noqa: E402
from paper_2406_18109_b200.executor import Executor, replay  # noqa: E402
from paper_2406_18109_b200.plan import PlanTrace  # noqa: E402

WANT = sys.argv[1:] or ["stencil_n1030_k1/fused", "stencil_n255_k2/fused", "cg_64x64_k1/fused", "bs_1e5_k1/fused",
                        "pcg_64x64_k2/fused"]


def main():
    with gzip.open(os.path.join(REPO, "tests", "golden", "plans_medium.json.gz"), "rt") as f:
        traces = {t["meta"]["name"]: PlanTrace.from_json(t) for t in json.load(f)["traces"]}
    bad = 0
    for name in WANT:
        tr = traces[name]
        ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, device=0)
        try:
            replay(ex, tr.events)
            got = {s: ex.get(s) for s in tr.live}
        finally:
            ex.close()
        ref = oracle_replay(tr)
        ok = all(np.allclose(got[s], ref.get(s), rtol=1e-12, atol=1e-12) for s in tr.live)
        bad += not ok
        print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
