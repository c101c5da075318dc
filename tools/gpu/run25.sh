cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "DK_K3_STAGES=2" "DK_K3_STAGES=3" "DK_K3_STAGES=4" "DK_K3_STAGES=2 DK_JIT_MINB=4" "DK_K3_STAGES=3 DK_JIT_MINB=4" "DK_K3_STAGES=4 DK_JIT_MINB=4" "DK_K3_STAGES=4 DK_JIT_MINB=3" "DK_JIT_MINB=2"; do
    R=$(env $cfg timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
    echo "cfg=[$cfg] $R"
done
done
for cfg in "" "DK_JIT_MINB=4"; do
    R=$(env $cfg timeout 600 python bench.py --workload bs --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
    echo "cfg=[$cfg] bs $R"
done
