cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu9.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu9.log
/usr/bin/time -v timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo bench=$?
grep -E "Elapsed|Maximum resident" gpurun_out/bench9.err
