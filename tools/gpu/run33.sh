cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
for v in "X=1" "DK_JIT_ROWS=1" "DK_JIT_MINB=6" "DK_JIT_MINB=8" "DK_JIT_UNROLL=4" "DK_JIT_UNROLL=4 DK_JIT_MINB=8" "DK_JIT_UNROLL=8"; do run stencil "$v"; done
run stencil X=1; run stencil DK_JIT_ROWS=1
run bs X=1; run cg X=1
