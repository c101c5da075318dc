cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants" 2>&1 | tail -3
for i in 1 2; do run stencil X=1; run stencil DK_K3_WS=1; done
run stencil "DK_K3_WS=1 DK_K3_STAGES=4"; run stencil "DK_K3_WS=1 DK_JIT_MINB=4"; run stencil "DK_K3_WS=1 DK_K3_TR=16 DK_K3_STAGES=2"
run stencil "DK_K3_WS=1 DK_K3_TR=12"
