cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 1500 $T bench.py --gpus 4 > gpurun_out/bench57_n4.json 2> gpurun_out/bench57_n4.err; echo bench4=$?
timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
