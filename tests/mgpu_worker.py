"""torchrun worker: golden multi-point plans on N real GPUs (NCCL), compared on rank 0.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_worker.py
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from conftest import golden_arrays, load_golden, same_bits  # noqa: E402
from paper_2406_18109_b200.executor import Executor, replay  # noqa: E402
from paper_2406_18109_b200.plan import PlanTrace  # noqa: E402

NAMES = [
    "stencil/fused", "stencil/unfused", "blackscholes_chain/fused", "blackscholes_chain/unfused",
    "jacobi/fused", "cg_like/fused", "cg_like/unfused",
    "stencil_bands_n8_k2/fused", "stencil_bands_n8_k2/unfused", "stencil_bands_n6_k4/fused",
    "cg_csr_8x8_k2/fused", "cg_csr_6x12_k4/fused", "cg_csr_6x12_k4/unfused", "pcg_csr_8x8_k2/fused",
] + [f"edge_{e}/{c}" for e in ("ragged_1d", "empty_tiles", "ragged_2d", "rank0", "nan_inf") for c in ("fused", "unfused")]


def gpusession_drop_in(rank, world, local):
    """GpuSession (reference front end + this backend) on `world` GPUs vs the reference Session on CPU."""
    ref = os.path.join(os.path.dirname(HERE), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "diffusekit")):
        return []
    sys.dont_write_bytecode = True
    sys.path.insert(0, ref)
    from diffusekit.pipeline import Session, SessionConfig, run_events
    from diffusekit.trace import gen_benchmark

    from paper_2406_18109_b200.session import GpuSession

    bad = []
    for name, kw in [("cg_like", dict(size=64, nodes=world * 2, iters=4)),
                     ("blackscholes_chain", dict(size=4096 * world, nodes=world, iters=5)),
                     ("jacobi", dict(size=32, nodes=world, iters=3))]:
        s = GpuSession(SessionConfig(), rank=rank, world=world, device=local)
        s.executor._comm = True  # communicator already initialised in this process
        s.executor.enable_p2p()
        rep = run_events(s, gen_benchmark(name, **kw))
        got = {sid: s.heap.get(sid) for sid in s.live_store_ids()}
        s.executor.close()
        if rank == 0:
            r = Session(SessionConfig())
            rep_ref = run_events(r, gen_benchmark(name, **kw))
            if rep.fused_prefixes != rep_ref.fused_prefixes:
                bad.append((f"gpusession/{name}", "plan"))
            for sid, g in got.items():
                w = r.heap.get(sid)
                if not (same_bits(g, w) or np.allclose(g, w, rtol=1e-12, atol=1e-12 * max(1.0, float(np.abs(w).max())))):
                    bad.append((f"gpusession/{name}", sid))
    return bad


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cases = {c["name"]: c for c in load_golden("bench_small.json.gz") + load_golden("fuzz250.json.gz")}
    names = NAMES + [f"fuzz{s}/fused" for s in range(0, 250, 5)]
    bad, moved, exact, close, p2p_folds = [], 0, 0, 0, 0
    uid = None
    for name in names:
        case = cases[name]
        tr = PlanTrace.from_json(case["trace"])
        ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, rank=rank, world=world,
                      device=local)
        if uid is None:
            obj = [ex.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ex.init_comm(obj[0])
            uid = True
        else:
            ex._comm = True
            ex.enable_p2p()
        replay(ex, tr.events)
        got = {s: ex.get(s) for s in tr.live}
        moved += ex.stats.transfers
        p2p_folds += ex.stats.p2p_folds
        ex.close()
        if rank == 0:
            for s, w in golden_arrays(case).items():
                if same_bits(got[s], w):
                    exact += 1
                elif np.allclose(got[s], w, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(w))))):
                    close += 1
                else:
                    bad.append((name, s))
    bad += gpusession_drop_in(rank, world, local)
    consumed = 0
    if os.environ.get("DK_P2P", "1") == "1":
        # the SpMV + partial-dot epilogue across GPUs: p.q rides in the next window's board block
        for name in ("cg_csr_8x8_k2/fused", "cg_csr_6x12_k4/fused", "pcg_csr_8x8_k2/fused"):
            case = cases[name]
            tr = PlanTrace.from_json(case["trace"])
            ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, rank=rank, world=world,
                          device=local, fuse_spmv_dot=True)
            ex._comm = True
            ex.enable_p2p()
            replay(ex, tr.events)
            got = {s: ex.get(s) for s in tr.live}
            st = dict(ex.spmv_dot_stats)
            ex.close()
            consumed += st["consumed"]
            # every rank must own a point of the SpMV for the epilogue to be used across GPUs
            spmv_vol = max(e.task.volume for e in tr.execs() if e.task.kind == "SPMV_CSR")
            if st["consumed"] != st["spmv"] or (spmv_vol >= world and st["consumed"] < 3):
                bad.append((f"spmv_dot/{name}", str(st)))
            if rank == 0:
                for s, w in golden_arrays(case).items():
                    if not np.allclose(got[s], w, rtol=1e-12, atol=1e-12 * max(1.0, float(np.max(np.abs(w))))):
                        bad.append((f"spmv_dot/{name}", s))
    if os.environ.get("DK_P2P", "1") == "1" and consumed == 0:
        bad.append(("spmv_dot", "never used"))
    if rank == 0:
        print(f"MGPU world={world} cases={len(names)} stores exact={exact} within_rtol={close} bad={bad[:8]} transfers={moved} "
              f"p2p_folds={p2p_folds} spmv_dot_consumed={consumed} (DK_P2P={os.environ.get('DK_P2P', '1')})")
        if bad:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
