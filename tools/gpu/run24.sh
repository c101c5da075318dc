cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "DK_K3_STAGES=2" "DK_K3_STAGES=3" "DK_K3_STAGES=4" "DK_K3_STAGES=4 DK_JIT_MINB=4"; do
    R=$(env $cfg timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['hbm_gbs_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'])")
    echo "cfg=[$cfg] stencil $R"
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "medium or golden_bench" 2>&1 | tail -1
