cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
runN() { R=$(env $3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $2 --workload $1 --steps 40 --warmup 5 --quick 2>gpurun_out/err_$1_$2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ranks_ms_per_step'], d['host_enqueue_ms_per_step'])"); echo "N$2 $1 $3 $R"; }
for i in 1 2 3; do runN cg 2 X=1; runN cg 2 DK_MPLAN=0; done
for i in 1 2; do runN cg 2 DK_P2P=0; runN cg 2 "DK_P2P=0 DK_MPLAN=0"; done
