cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/gpu/mixprobe.py 2>&1 | grep add
for v in "TAG=default" "DK_JIT_PREFETCH=1" "DK_JIT_PREFETCH=1 DK_JIT_UNROLL=1" "DK_JIT_PREFETCH=1 DK_JIT_UNROLL=1 DK_JIT_MINB=6"; do
env TAG="$v" $v timeout 300 python tools/gpu/jitprobe.py 2>&1 | tail -2
done
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
for w in bs stencil cg; do run $w X=1; run $w DK_JIT_PREFETCH=1; done
DK_JIT_PREFETCH=1 timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
