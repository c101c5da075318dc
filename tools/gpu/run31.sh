cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for i in 1 2; do
for v in "X=1" "DK_JIT_NO_H=1" "DK_JIT_MINB=6" "DK_JIT_MINB=8"; do
R=$(env $v timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
echo "$v stencil $R"
done; done
