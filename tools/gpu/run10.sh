cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
START=$(date +%s)
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo bench=$? elapsed=$(( $(date +%s) - START ))s
tail -3 gpurun_out/bench10.err
