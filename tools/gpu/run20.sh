cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu20.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu20.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo bench=$?
