cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu16.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu16.log
