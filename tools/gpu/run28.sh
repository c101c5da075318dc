cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29531 tests/mgpu_worker.py > gpurun_out/mgpu28.log 2>&1; echo mgpu=$?
grep MGPU gpurun_out/mgpu28.log; grep -iE "error|Traceback" gpurun_out/mgpu28.log | head -5
