# 4 GPUs: is the per-rank imbalance (stencil ranks 2/3 slower after the BS runs) reproducible?
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29550
runN() { P=$((P+1)); R=$(env $3 timeout 300 $TR --master-port $P bench.py --gpus 4 --workload $1 --steps 20 --warmup 3 --quick --pre "$2" 2>>gpurun_out/err71.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('ranks_ms_per_step'), d.get('host_enqueue_ms_per_step'), d['per_exec_ms'])"); echo "wl=$1 pre=[$2] env=$3 $R"; }
nvidia-smi topo -m
runN stencil "" X=1
runN stencil "" X=1
runN stencil "bs,bs:unfused" X=1
runN stencil "" DK_P2P=0
runN cg "" X=1
runN cg "stencil,stencil:unfused" X=1
runN cg "" DK_P2P=0
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv
