cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in stencil bs cg pcg; do
    R=$(timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['per_exec_ms'])")
    echo "$wl $R"
done
