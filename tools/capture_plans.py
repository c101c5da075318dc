"""Record the unchanged reference front end's plans for the benchmark workloads.

    python tools/capture_plans.py            # writes paper_2406_18109_b200/workloads/*.json.gz
                                             # and tests/golden/plans_medium.json.gz

Analysis never touches data (``SessionConfig(execute=False)``), so full-size
configurations (1e9 options, 32768^2 bands, 67M-row CG) are captured in
seconds.  The GPU box replays these traces; it has no copy of the reference.
"""

from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

from refcapture import import_reference, record_events  # noqa: E402

import_reference()
from diffusekit.pipeline import SessionConfig  # noqa: E402

import workloads as W  # noqa: E402

OUT = os.path.join(REPO, "paper_2406_18109_b200", "workloads")
ITERS = 24


def gens(N: int):
    return {
        "bs": lambda it: W.blackscholes(1_000_000_000 * N, N, it),
        "stencil": lambda it: W.stencil_bands(32768, N, it),
        "cg": lambda it: W.cg_csr(8192, 8192 * N, N, it),
        "pcg": lambda it: W.pcg_csr(8192, 8192 * N, N, it),
    }


def capture(name, gen, iters, fused, execute=False):
    events, init, dtypes = gen(iters)
    cfg = SessionConfig(execute=execute, fusion=fused)
    _, report, trace = record_events(events, cfg, init=init)
    trace.dtypes = dict(dtypes)
    trace.meta["name"] = name
    trace.meta["fused"] = fused
    return trace


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--large-only" in sys.argv:
        large()
        return
    if "--multirank-only" in sys.argv:
        multirank()
        return
    if "--medium-only" not in sys.argv:
        full_size()
    medium()
    large()
    multirank()


def multirank():
    """Eight-point plans for the world-4 / world-8 gloo tests (tests/test_multirank_gloo.py):
    one or two launch points per rank, compared with the oracle there."""
    out = []
    for name, gen, iters in [
        ("stencil_bands_n4_k8", lambda it: W.stencil_bands(4, 8, it), 3),
        ("cg_csr_8x16_k8", lambda it: W.cg_csr(8, 16, 8, it), 4),
        ("pcg_csr_8x16_k8", lambda it: W.pcg_csr(8, 16, 8, it), 4),
        # one tile per rank at world 4 with interior rows (t = 64 > 2 nx): the overlapped-halo SpMV
        ("cg_csr_4x64_k4", lambda it: W.cg_csr(4, 64, 4, it), 4),
        ("pcg_csr_4x64_k4", lambda it: W.pcg_csr(4, 64, 4, it), 4),
    ]:
        for fused in (True, False):
            tr = capture(f"{name}/{'fused' if fused else 'unfused'}", gen, iters, fused)
            out.append(tr.to_json())
    with gzip.open(os.path.join(REPO, "tests", "golden", "plans_k8.json.gz"), "wt", compresslevel=9) as f:
        json.dump({"format": "dk-plans-1", "traces": out}, f, separators=(",", ":"))
    print("k8 traces:", len(out))


def large():
    """Multi-band plans at large size for the one-GPU full-size parity tests (tests/test_gpu_fullsize.py):
    four 8192^2 bands on one GPU (four launch points per launch)."""
    out = []
    for fused in (True, False):
        tr = capture(f"stencil_8192_k4/{'fused' if fused else 'unfused'}", lambda it: W.stencil_bands(8192, 4, it),
                     12 if fused else 6, fused)
        out.append(tr.to_json())
    with gzip.open(os.path.join(REPO, "tests", "golden", "plans_large.json.gz"), "wt", compresslevel=9) as f:
        json.dump({"format": "dk-plans-1", "traces": out}, f, separators=(",", ":"))
    print("large traces:", len(out))


def full_size():
    for N in (1, 2, 4, 8):
        for wl, gen in gens(N).items():
            iters = ITERS + (4 if wl == "bs" else 0)
            for fused in (True, False):
                name = f"{wl}_{'fused' if fused else 'unfused'}_n{N}"
                tr = capture(name, gen, iters, fused)
                tr.meta["gpus"] = N
                tr.save(os.path.join(OUT, name + ".json.gz"))
                print(name, tr.meta["report"]["fused_prefixes"][-6:], len(tr.events))
    # C1: the reference's own CPU case (1M options, one partition) -- CPU baseline sample
    for fused in (True, False):
        name = f"bs_{'fused' if fused else 'unfused'}_c1"
        tr = capture(name, lambda it: W.blackscholes(1_000_000, 1, it), ITERS + 4, fused)
        tr.save(os.path.join(OUT, name + ".json.gz"))
        print(name, tr.meta["report"]["fused_prefixes"][-3:])
    # bounded CPU-baseline samples of the other workloads (one partition)
    for wl, gen in {
        "stencil": lambda it: W.stencil_bands(2048, 1, it),
        "cg": lambda it: W.cg_csr(1024, 1024, 1, it),
        "pcg": lambda it: W.pcg_csr(1024, 1024, 1, it),
    }.items():
        for fused in (True, False):
            name = f"{wl}_{'fused' if fused else 'unfused'}_cpu"
            tr = capture(name, gen, 12, fused)
            tr.save(os.path.join(OUT, name + ".json.gz"))


def medium():
    # medium sizes for GPU-vs-oracle parity tests (traces only; the oracle runs on the box)
    med = []
    for name, gen in [
        ("bs_1e5_k1", lambda: W.blackscholes(100_000, 1, 6)),
        ("bs_1e5_k2", lambda: W.blackscholes(100_000, 2, 6)),
        ("stencil_n256_k1", lambda: W.stencil_bands(256, 1, 3)),
        ("stencil_n255_k2", lambda: W.stencil_bands(255, 2, 3)),
        # row widths around the warp / CTA / pair boundaries of the JIT's row loop
        ("stencil_n34_k1", lambda: W.stencil_bands(34, 1, 2)),
        ("stencil_n67_k1", lambda: W.stencil_bands(67, 1, 2)),
        ("stencil_n1030_k1", lambda: W.stencil_bands(1030, 1, 2)),
        ("stencil_n1027_k3", lambda: W.stencil_bands(1027, 3, 2)),
        ("cg_64x64_k1", lambda: W.cg_csr(64, 64, 1, 8)),
        ("cg_64x64_k2", lambda: W.cg_csr(64, 64, 2, 8)),
        ("pcg_64x64_k2", lambda: W.pcg_csr(64, 64, 2, 8)),
        ("cg_64x128_k4", lambda: W.cg_csr(64, 128, 4, 6)),
    ]:
        for fused in (True, False):
            tr = capture(f"{name}/{'fused' if fused else 'unfused'}", lambda it, g=gen: g(), 0, fused)
            med.append(tr.to_json())
    with gzip.open(os.path.join(REPO, "tests", "golden", "plans_medium.json.gz"), "wt", compresslevel=9) as f:
        json.dump({"format": "dk-plans-1", "traces": med}, f, separators=(",", ":"))
    print("medium traces:", len(med))


if __name__ == "__main__":
    main()
