"""torchrun worker: the peer-memory protocols under rank skew (2+ GPUs).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_stress.py

Replays the one-tile-per-rank CG plan (``plans_k8.json.gz`` ``cg_csr_4x64_k4`` at world 4, the
golden ``cg_csr_8x8_k2`` at world 2) for many cycled iterations -- every iteration two reductions
through the epoch-tagged peer boards and one SpMV halo through the copy-engine mailboxes -- while
each rank sleeps a random 0-2 ms before random launches, so ranks run up to several board epochs
and mailbox messages apart.  A broken ring or mailbox invariant traps (flags carry the epoch's tag);
a silently wrong fold shows up as a result that differs from the same stream run on rank 0's GPU
alone (world 1): the point-order fold makes the two bit-identical.
"""

import gzip
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from conftest import GOLDEN, load_golden, same_bits  # noqa: E402
from paper_2406_18109_b200.executor import Executor  # noqa: E402
from paper_2406_18109_b200.plan import PlanTrace  # noqa: E402

CYCLES = int(os.environ.get("DK_STRESS_CYCLES", "40"))


def _trace(world):
    if world == 2:
        return PlanTrace.from_json({c["name"]: c for c in load_golden("bench_small.json.gz")}["cg_csr_8x8_k2/fused"]["trace"])
    with gzip.open(os.path.join(GOLDEN, "plans_k8.json.gz"), "rt") as f:
        tr = {t["meta"]["name"]: t for t in json.load(f)["traces"]}
    return PlanTrace.from_json(tr["cg_csr_4x64_k4/fused"])


def _run(ex, tr, its, seq, jitter, rng):
    for i in seq:
        # fresh reduction targets each cycled iteration (bench.fresh_targets)
        for k, e in its[i]:
            if k == "exec":
                for a in e.task.args:
                    if a.reduces and tr.shapes.get(a.store) == () and a.store in ex.stores:
                        ex.free(a.store)
        for k, e in its[i]:
            if k == "exec":
                if jitter and rng.random() < 0.3:
                    time.sleep(rng.uniform(0, 2e-3))
                ex.execute(e.task, e.kernel, e.temp_positions)
            elif k == "free":
                ex.free(e)
    ex.sync()


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    tr = _trace(world)
    its = tr.iterations()
    sig = [tuple(e.f for k, e in it if k == "exec") for it in its]
    steady = next(i for i in range(len(its)) if sig[i] == sig[-1])
    seq = list(range(steady)) + [steady + (c % (len(its) - steady)) for c in range(CYCLES)]
    ex = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, rank=rank, world=world, device=local)
    obj = [ex.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ex.init_comm(obj[0])
    assert ex._p2p, "peer boards not enabled"
    _run(ex, tr, its, seq, True, random.Random(1000 + rank))
    got = {s: ex.get(s) for s in tr.live if s in ex.stores}
    stats = dict(vars(ex.stats))
    ex.close()
    bad = []
    if rank == 0:
        ref = Executor(shapes=tr.shapes, seed=tr.seed, init=tr.init, dtypes=tr.dtypes, rank=0, world=1, device=local)
        _run(ref, tr, its, seq, False, random.Random(0))
        for s, g in got.items():
            if s in ref.stores and not same_bits(g, ref.get(s)):
                bad.append(s)
        ref.close()
        print(f"STRESS world={world} iterations={len(seq)} p2p_folds={stats['p2p_folds']} p2p_halos={stats['p2p_halos']} "
              f"compared={len(got)} bad={bad[:8]}")
        if bad or stats["p2p_folds"] < CYCLES:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
