"""Time single JIT kernels on torch-allocated 1-D f64 buffers (1e9 elements):
a plain x+y (the 2-read/1-write mix of the BS window) and the BS window itself."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2406_18109_b200 import runtime as rt  # noqa: E402
from paper_2406_18109_b200.plan import PlanTrace  # noqa: E402

lib = rt.load()
rt.check(lib.dk_init(0))
n = int(os.environ.get("N", 1_000_000_000))
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.rand(n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
s = torch.cuda.Stream()  # a real stream: dk_set_stream(0) would mean the library's own
torch.cuda.set_stream(s)
rt.check(lib.dk_set_stream(s.cuda_stream))

tr = PlanTrace.load(os.path.join(os.path.dirname(rt.HERE), "paper_2406_18109_b200", "workloads", "bs_fused_n1.json.gz"))
big = [e for e in tr.execs() if e.kernel is not None and len(e.kernel.slots) == 3 and e.f > 10][0]
progs = {
    "add": ("DK1 3 0 0 1\nslot 0 1 P R\nslot 1 1 P R\nslot 2 1 P W\nnest 2 1 1\n S 2 0 (B + (L 0 0) (L 1 0))\nend\n", ()),
    "bs": (big.kernel.wire([sl.decl_rank for sl in big.kernel.slots]), big.task.scalars),
}
views = (rt.dk_view * 3)()
for i, t in enumerate((x, y, z)):
    views[i].ptr, views[i].rank, views[i].dtype = t.data_ptr(), 1, 0
    views[i].ext[0], views[i].stride[0] = n, 1
for name, (text, sc) in progs.items():
    h = ctypes.c_int64()
    b = text.encode()
    rt.check(lib.dk_kernel_compile(b, len(b), ctypes.byref(h)))
    scal = (ctypes.c_double * max(1, len(sc)))(*sc)

    def go():
        rt.check(lib.dk_launch(h, views, 3, scal, len(sc), 0))

    for _ in range(3):
        go()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(8):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); go(); e.record(); e.synchronize()
        best = min(best, a.elapsed_time(e))
    print(f"{name} {os.environ.get('TAG', '')}: {best:.3f} ms  {24 * n / best / 1e6:.0f} GB/s")
