cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench18.json 2> gpurun_out/bench18.err; echo bench=$?
tail -3 gpurun_out/bench18.err
