cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in bs stencil cg pcg; do
    R=$(timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['hbm_gbs_step'])")
    echo "$wl $R"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
