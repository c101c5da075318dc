cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi topo -m | head -6
timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 1500 $T bench.py --gpus 4 > gpurun_out/bench52_n4.json 2> gpurun_out/bench52_n4.err; echo bench4=$?
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
timeout 1500 $T2 bench.py --gpus 2 > gpurun_out/bench52_n2.json 2> gpurun_out/bench52_n2.err; echo bench2=$?
timeout 600 $T bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > gpurun_out/bench52_ref4.json 2> gpurun_out/bench52_ref4.err; echo ref4=$?
