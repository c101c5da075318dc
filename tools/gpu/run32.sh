cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in stencil bs; do
for h in "X=1" "DK_JIT_NO_H=1"; do
for u in 2 4 8; do
for m in 4 6 8; do
R=$(env $h DK_JIT_UNROLL=$u DK_JIT_MINB=$m timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
echo "$wl $h U=$u M=$m $R"
done; done
[ $wl = bs ] && break
done; done
