cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/pytest_mgpu4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_mgpu4.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2951$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench6_n$N.json 2> gpurun_out/bench6_n$N.err; echo bench$N=$?
done
