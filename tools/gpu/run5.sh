cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29511 tests/mgpu_worker.py > gpurun_out/mgpu2.log 2>&1; echo mgpu=$?
tail -5 gpurun_out/mgpu2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench5_n2.json 2> gpurun_out/bench5_n2.err; echo bench2=$?
tail -3 gpurun_out/bench5_n2.err
