cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
run bs X=1; run bs X=1; run stencil X=1; run cg X=1; run bs DK_JIT_MINB=4
