cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench58.json 2> gpurun_out/bench58.err; echo bench=$?
tail -c 1500 gpurun_out/bench58.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench58_ref.json 2>gpurun_out/bench58_ref.err; echo ref=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
