cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu55.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu55.log
run1() { R=$(env $2 CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['host_enqueue_ms_per_step'], d['per_exec_ms'])"); echo "N1 $1 $2 $R"; }
runN() { R=$(env $3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $2 --workload $1 --steps 20 --warmup 3 --quick 2>gpurun_out/err_$1_$2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ranks_ms_per_step'], d['host_enqueue_ms_per_step'])"); echo "N$2 $1 $3 $R"; }
for w in cg pcg stencil bs; do run1 $w X=1; done
run1 cg DK_MPLAN=0
for w in cg pcg stencil bs; do runN $w 2 X=1; done
runN cg 2 DK_MPLAN=0
