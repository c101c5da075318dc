cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi topo -m | head -5
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
run() { R=$(env $2 timeout 600 $T bench.py --gpus 2 --workload $1 --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_exec_ms'])"); echo "$1 $2 $R"; }
for i in 1 2; do run cg DK_P2P=1; run cg DK_P2P=0; done
run pcg DK_P2P=1; run pcg DK_P2P=0
run stencil DK_P2P=1; run stencil DK_P2P=0
run bs DK_P2P=1
