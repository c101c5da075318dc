# 4 GPUs at HEAD: full default bench line, then CG alone vs CG after the other workloads
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29541 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo n4=$?
runN() { R=$(env $3 timeout 300 $TR --master-port $4 bench.py --gpus 4 --workload cg --steps 20 --warmup 3 --quick --pre "$2" 2>>gpurun_out/err70.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('ranks_ms_per_step'), d.get("host_enqueue_ms_per_step"), d['per_exec_ms'])"); echo "pre=[$2] $3 $R"; }
runN "" X=1 29542
runN "bs:unfused" X=1 29543
runN "stencil" X=1 29544
runN "" DK_P2P=0 29545
