cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
for w in stencil bs cg pcg; do run $w X=1; run $w DK_JIT_PERSIST=1; done
for v in "DK_JIT_MINB=4" "DK_JIT_MINB=8" "DK_JIT_UNROLL=1" "DK_JIT_UNROLL=4"; do run stencil "$v"; run bs "$v"; done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
