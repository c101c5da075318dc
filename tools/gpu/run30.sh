cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do
for v in 0 1; do
if [ $v = 1 ]; then export DK_JIT_NO_SHIFT=1; else unset DK_JIT_NO_SHIFT; fi
R=$(timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
echo "noshift=$v stencil $R"
done; done
