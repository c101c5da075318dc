cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { R=$(env $2 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants" 2>&1 | tail -3
run stencil X=1; run stencil DK_K3S=1
for pf in 2 4 6; do run stencil "DK_K3S=1 DK_K3S_PF=$pf"; done
for rb in 32 128 256; do run stencil "DK_K3S=1 DK_K3S_RB=$rb"; done
run stencil "DK_K3S=1 DK_JIT_MINB=3"; run stencil "DK_K3S=1 DK_JIT_MINB=5 DK_K3S_PF=2"
run stencil "DK_K3S=1 DK_JIT_RWAVES=8"; run stencil "DK_K3S=1 DK_JIT_RWAVES=2"
run stencil X=1; run stencil DK_K3S=1
