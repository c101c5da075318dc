cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "medium or nan or pcg64_init" > gpurun_out/plain21.log 2>&1; echo plain=$?
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -k "medium or nan or pcg64_init" > gpurun_out/memcheck21.log 2>&1; echo memcheck=$?
tail -15 gpurun_out/memcheck21.log
