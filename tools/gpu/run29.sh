cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for wl in stencil cg bs; do
R=$(timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29541 bench.py --gpus 2 --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
echo "N=2 $wl $R"
R=$(timeout 900 python bench.py --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['per_exec_ms'])")
echo "N=1 $wl $R"
done
