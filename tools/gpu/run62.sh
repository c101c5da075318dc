cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
runN() { R=$(env $3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload cg --steps 20 --warmup 3 --quick --pre "$2" 2>gpurun_out/err62.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ranks_ms_per_step'], d['per_exec_ms'])"); echo "pre=[$2] $3 $R"; }
runN "" X=1
runN "bs" X=1
runN "stencil" X=1
runN "bs:unfused" X=1
runN "stencil:unfused" X=1
runN "stencil" DK_VA_POOL_GB=0
runN "stencil" DK_P2P=0
runN "stencil" DK_MPLAN=0
runN "cg" X=1
