"""B200-native execution backend for Diffuse fused tasks (arXiv 2406.18109).

The reference front end (``diffusekit``: windowing, scale-free fusion
analysis, temporaries, memoization, kernel composition) stays unchanged; this
package replaces what runs once a fused window has been formed:

* ``executor.Executor`` -- device heap + launch engine (one GPU per process),
  partition -> GPU mapping and inter-GPU coherence;
* ``csrc/`` -- ``libdk_b200.so``: VMM-backed stores, the NVRTC JIT that turns
  a fused kernel into one sm_100a kernel, reductions, builtins, NCCL moves;
* ``session.GpuSession`` -- drop-in ``diffusekit.Session`` subclass;
* ``plan`` -- recorded front-end decisions replayed where the reference is
  not installed (the GPU box).

Heavy pieces are imported lazily: ``import paper_2406_18109_b200`` does not
load CUDA.
"""

from .ir import KProg, TaskDesc, lower_kernel, lower_task, rect_of  # noqa: F401
from .plan import ExecStep, PlanTrace  # noqa: F401

__version__ = "0.1.0"


def executor(**kw):
    """Create an :class:`executor.Executor` (loads ``libdk_b200.so``)."""
    from .executor import Executor

    return Executor(**kw)
