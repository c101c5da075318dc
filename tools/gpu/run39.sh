cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
for rw in 1 2 4 8 16; do run cg DK_JIT_RWAVES=$rw; done
run pcg DK_JIT_RWAVES=1; run pcg DK_JIT_RWAVES=4
run cg DK_JIT_PERSIST=1
for u in 2 4 8; do for m in 4 6 8; do run bs "DK_JIT_UNROLL=$u DK_JIT_MINB=$m"; run stencil "DK_JIT_UNROLL=$u DK_JIT_MINB=$m"; done; done
