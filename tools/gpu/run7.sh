cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu7.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu7.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29522 bench.py --gpus 2 --workload cg --steps 10 --warmup 3 > gpurun_out/bench7_cg2.json 2> gpurun_out/bench7_cg2.err; echo bench=$?
