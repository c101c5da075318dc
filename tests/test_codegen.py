"""Device-free checks of the JIT: generated CUDA for recorded reference kernels compiles with NVRTC for sm_100a."""

import ctypes

import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def rt():
    from paper_2406_18109_b200.build import build

    build()
    try:
        ctypes.CDLL("libcuda.so.1", mode=ctypes.RTLD_GLOBAL)
    except OSError:
        ctypes.CDLL("/usr/local/cuda/lib64/stubs/libcuda.so", mode=ctypes.RTLD_GLOBAL)
    from paper_2406_18109_b200 import runtime

    runtime.load()
    return runtime


def views_for(rt, task, kp, shapes, point=None):
    from paper_2406_18109_b200.ir import rect_of

    p = point or tuple(0 for _ in task.launch)
    views = (rt.dk_view * len(kp.slots))()
    base = 1 << 32
    for i, s in enumerate(kp.slots):
        a = task.args[s.arg]
        shape = shapes[a.store]
        lo, hi = rect_of(shape, a.part, p)
        strides = [1] * len(shape)
        for d in range(len(shape) - 2, -1, -1):
            strides[d] = strides[d + 1] * shape[d + 1]
        v = views[i]
        v.ptr = base * (a.store + 1) + 8 * sum(l * st for l, st in zip(lo, strides))  # one base per store
        v.rank = len(shape)
        v.dtype = 0
        for d in range(len(shape)):
            v.ext[d] = hi[d] - lo[d]
            v.stride[d] = strides[d]
    return views


def codegen(rt, kp, views, compile_=True, scalars=()):
    text = kp.wire([s.decl_rank for s in kp.slots]).encode()
    n = ctypes.c_int64()
    sc = (ctypes.c_double * max(len(scalars), 1))(*scalars) if scalars else None
    rt.check(rt._lib.dk_kernel_codegen(text, len(text), views, len(kp.slots), sc, 1 if compile_ else 0, None, 0,
                                       ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    rt.check(rt._lib.dk_kernel_codegen(text, len(text), views, len(kp.slots), sc, 0, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def test_bench_kernels_compile(rt, tmp_path, monkeypatch):
    from paper_2406_18109_b200.plan import PlanTrace

    monkeypatch.setenv("DK_JIT_CACHE", str(tmp_path))
    seen = set()
    for case in load_golden("bench_small.json.gz"):
        tr = PlanTrace.from_json(case["trace"])
        for e in tr.execs():
            if e.kernel is None:
                continue
            key = e.kernel.wire([0] * len(e.kernel.slots))
            if key in seen:
                continue
            seen.add(key)
            src = codegen(rt, e.kernel, views_for(rt, e.task, e.kernel, tr.shapes))
            assert "__dadd_rn" in src or "dk_" in src
    assert len(seen) >= 20


def test_fused_blackscholes_kernel_is_one_register_nest(rt):
    from paper_2406_18109_b200.plan import PlanTrace

    case = {c["name"]: c for c in load_golden("bench_small.json.gz")}["blackscholes_chain/fused"]
    tr = PlanTrace.from_json(case["trace"])
    big = [e for e in tr.execs() if e.f == 67][0]
    src = codegen(rt, big.kernel, views_for(rt, big.task, big.kernel, tr.shapes), compile_=False,
                  scalars=big.task.scalars)
    body = src[src.index("__global__"):]
    assert body.count("__global__") == 1
    # 66 SetTemps per lane live in registers; only x, y are loaded and out stored,
    # as 16-byte aligned pairs
    assert body.count("dk_ld_A(") == 2 and body.count("dk_st_A(") == 1
    assert "dk_ld_C(" not in body and "dk_st_C(" not in body
    assert "dk_mul(" in body and "dk_neg(" in body
    # 26 task scalars, two distinct values: only two parameter slots are read
    assert sorted(set(body.split("P.sc[")[i].split("]")[0] for i in range(1, body.count("P.sc[") + 1))) == ["0", "1"]


def test_privilege_violation_detected_without_device(rt):
    from paper_2406_18109_b200.errors import PrivilegeError
    from paper_2406_18109_b200.ir import ArgDesc, KProg, PartDesc, Slot, TaskDesc

    tile = PartDesc("tiling", (4,), (0,), ((1,),), (0,))
    kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "R", 1)), (), 0,
               ((1, 1, (("store", 1, (0,), ("ld", 0, (0,))),)),), False)
    task = TaskDesc("COPY", (2,), (ArgDesc(0, tile, "R"), ArgDesc(1, tile, "R")))
    with pytest.raises(PrivilegeError):
        codegen(rt, kp, views_for(rt, task, kp, {0: (8,), 1: (8,)}), compile_=False)


def test_offset_out_of_bounds_detected(rt):
    from paper_2406_18109_b200.errors import BoundsError
    from paper_2406_18109_b200.ir import ArgDesc, KProg, PartDesc, Slot, TaskDesc

    tile = PartDesc("tiling", (4,), (0,), ((1,),), (0,))
    kp = KProg((Slot("a0", 0, False, "R", 1), Slot("a1", 1, False, "W", 1)), (), 0,
               ((1, 1, (("store", 1, (0,), ("ld", 0, (1,))),)),), False)
    task = TaskDesc("SHIFT", (2,), (ArgDesc(0, tile, "R"), ArgDesc(1, tile, "W")))
    with pytest.raises(BoundsError):
        codegen(rt, kp, views_for(rt, task, kp, {0: (8,), 1: (8,)}), compile_=False)


def test_odd_parity_pair_variants(rt, monkeypatch):
    """Stencil COPY work -> grid interior (the interior view starts one element
    past a 16-byte boundary).  Default: one CTA per chunk of pairs (no
    persistent grid-stride loop), aligned 16-byte loads, split 8-byte stores.
    DK_JIT_H: the target moves as aligned pairs shifted by one
    element, completed by a warp shuffle ('H')."""
    from paper_2406_18109_b200.plan import PlanTrace

    case = {c["name"]: c for c in load_golden("bench_small.json.gz")}["stencil/fused"]
    tr = PlanTrace.from_json(case["trace"])
    copy = [e for e in tr.execs() if e.f == 1][0]
    win = [e for e in tr.execs() if e.f == 5][0]

    def body(e):
        src = codegen(rt, e.kernel, views_for(rt, e.task, e.kernel, tr.shapes), scalars=e.task.scalars)
        return src[src.index("__global__"):]

    b = body(copy)
    assert "c < nchunks" in b and "dk_ld_A(" in b and "dk_st_C(" in b and "__shfl" not in b
    monkeypatch.setenv("DK_JIT_H", "1")
    b = body(copy)
    assert "__shfl_down_sync" in b and "dk_st_C(" not in b and "dk_ld_C(" not in b
    b = body(win)  # the window's shifted views (not TMA-staged at this size)
    assert "__shfl_up_sync" in b and "dk_ld_C(" not in b


def test_alias_corpus_kernels_compile(rt):
    """The aliasing / POW / copy-in kernels (alias_streams corpus) compile for sm_100a, incl. dk_pow."""
    from paper_2406_18109_b200 import aliasing
    from paper_2406_18109_b200.plan import PlanTrace

    seen = set()
    n_pow = 0
    for case in load_golden("alias_streams.json.gz"):
        tr = PlanTrace.from_json(case["trace"])
        for e in tr.execs():
            if e.kernel is None or e.kernel.wire([s.decl_rank for s in e.kernel.slots]) in seen:
                continue
            seen.add(e.kernel.wire([s.decl_rank for s in e.kernel.slots]))
            src = codegen(rt, e.kernel, views_for(rt, e.task, e.kernel, tr.shapes))
            n_pow += "dk_pow(" in src.split("__global__", 1)[-1]
    for r in (1, 2):
        kp = aliasing.copy_kprog(r)
        codegen(rt, kp, views_for(rt, _copy_task(r), kp, {0: (6,) * r, 1: (6,) * r}))
    assert n_pow >= 2


def _copy_task(rank):
    from paper_2406_18109_b200.ir import ArgDesc, PartDesc, TaskDesc

    ident = tuple(tuple(1 if i == j else 0 for j in range(rank)) for i in range(rank))
    p = PartDesc("tiling", (6,) * rank, (0,) * rank, ident, (0,) * rank)
    return TaskDesc("COPY", (1,) * rank, (ArgDesc(0, p, "R"), ArgDesc(1, p, "W")))


def test_multi_nest_windows_compile_as_one_kernel(rt):
    """Windows whose tasks iterate differently-shaped domains lower to several nests; every such
    kernel of the fuzz corpus is generated as ONE cooperative kernel (``_m``: each nest a device
    function over the same 256-thread CTAs, ``dk_grid_sync`` between nests) and compiles for sm_100a;
    DK_JIT_SPLIT_NESTS=1 restores one launch per nest."""
    import os

    from paper_2406_18109_b200.plan import PlanTrace

    seen = set()
    merged = 0
    for case in load_golden("fuzz250.json.gz")[::3]:
        tr = PlanTrace.from_json(case["trace"])
        for e in tr.execs():
            if e.kernel is None or len(e.kernel.nests) < 2:
                continue
            w = e.kernel.wire([s.decl_rank for s in e.kernel.slots])
            if w in seen:
                continue
            seen.add(w)
            src = codegen(rt, e.kernel, views_for(rt, e.task, e.kernel, tr.shapes), compile_=len(seen) <= 12)
            assert src.count("__global__") == 1 and "dk_m(" in src, src[-2000:]
            assert src.count("dk_grid_sync((unsigned*)P.gbar)") == len(e.kernel.nests) - 1
            merged += 1
    assert merged >= 20
    os.environ["DK_JIT_SPLIT_NESTS"] = "1"
    try:
        src = codegen(rt, e.kernel, views_for(rt, e.task, e.kernel, tr.shapes), compile_=False)
    finally:
        del os.environ["DK_JIT_SPLIT_NESTS"]
    assert src.count("__global__") == len(e.kernel.nests)


def test_multi_nest_merge_size_cap():
    """Nests above DK_JIT_MERGE_MAX elements keep one launch per nest (the saved launch is worth
    less than the one-wave grid-stride walk there): with a cap of 0 every non-empty multi-nest window splits."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import ctypes, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
from conftest import load_golden
import test_codegen as tc
from paper_2406_18109_b200.plan import PlanTrace
try:
    ctypes.CDLL("libcuda.so.1", mode=ctypes.RTLD_GLOBAL)
except OSError:
    ctypes.CDLL("/usr/local/cuda/lib64/stubs/libcuda.so", mode=ctypes.RTLD_GLOBAL)
from paper_2406_18109_b200 import runtime
runtime.load()
n = 0
for case in load_golden("fuzz250.json.gz")[::10]:
    tr = PlanTrace.from_json(case["trace"])
    for e in tr.execs():
        if e.kernel is not None and len(e.kernel.nests) > 1:
            src = tc.codegen(runtime, e.kernel, tc.views_for(runtime, e.task, e.kernel, tr.shapes), compile_=False)
            assert src.count("__global__") == len(e.kernel.nests), src[-500:]
            n += 1
print("split", n)
""" % (os.path.join(repo, "tests"), repo)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, DK_JIT_MERGE_MAX="0"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.split()[-1]) >= 5, r.stdout
