cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_streaming.py -q > gpurun_out/pytest_gpu17.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu17.log
