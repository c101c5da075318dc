"""Host-side cost of the executor per iteration (planning, coherence, ctypes
marshalling) with a no-op device: every dk_* call returns at once, so the time
measured is what the Python/C-ABI side adds on top of the GPU work.

    python tools/host_overhead.py [plan] [world]     (default: cg_fused_n4, every rank simulated in turn)

A rank whose host time per iteration exceeds its device time starves its GPU
(and, through the exchanges, every other rank).
"""

from __future__ import annotations

import ctypes
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2406_18109_b200.executor import Executor, replay  # noqa: E402
from paper_2406_18109_b200.plan import PlanTrace  # noqa: E402


class NullLib:
    """Accepts every C-ABI call; pointers are fake, nothing is computed."""

    def __init__(self):
        self.n = 0

    def _ok(self, *args):
        self.n += 1
        for a in args:
            # out-parameters (byref / pointers) get a plausible non-zero value
            if isinstance(a, ctypes._Pointer) or type(a).__name__ == "CArgObject":
                try:
                    a._obj.value = 1 << 20
                except (AttributeError, TypeError):
                    pass
        return 0

    def dk_p2p_init(self, ref):
        ref._obj.value = 1
        return 0

    def dk_kernel_num_reductions(self, h, ref):
        return 0

    def dk_pcg64_rejects(self, state, inc, draw_end, out, cap, n_out):
        n_out._obj.value = 0  # no rejection breakpoints
        return 0

    def __getattr__(self, name):
        if name.startswith("dk_"):
            return self._ok
        raise AttributeError(name)


def main():
    plan = sys.argv[1] if len(sys.argv) > 1 else "cg_fused_n4"
    tr = PlanTrace.load(os.path.join(REPO, "paper_2406_18109_b200", "workloads", plan + ".json.gz"))
    its = tr.iterations()
    world = int(sys.argv[2]) if len(sys.argv) > 2 else max(e.task.volume for e in tr.execs())
    for rank in range(world):
        ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, rank=rank, world=world,
                      lib=NullLib())
        ex._comm = True
        ex.enable_p2p()
        n_warm = len(its) // 2
        for it in its[:n_warm]:
            replay(ex, it)
        t0 = time.perf_counter()
        for it in its[n_warm:]:
            replay(ex, it)
        dt = (time.perf_counter() - t0) / (len(its) - n_warm)
        print(f"{plan} rank {rank}/{world}: host {dt * 1e3:.3f} ms per iteration")


if __name__ == "__main__":
    main()
