cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run1() { R=$(env $2 CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])"); echo "N1 $1 $2 $R"; }
runN() { R=$(env $3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $2 --workload $1 --steps 20 --warmup 3 --quick 2>gpurun_out/err_$1_$2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_exec_ms'])"); echo "N$2 $1 $3 $R"; }
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv_variants" 2>&1 | tail -2
for i in 1 2; do run1 cg X=1; run1 cg DK_SPMV_WARP=1; done
for i in 1 2; do runN cg 4 DK_P2P=1; runN cg 4 DK_P2P=0; done
runN pcg 4 DK_P2P=1; runN cg 2 DK_P2P=1; runN bs 4 X=1
