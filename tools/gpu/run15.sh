cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name --format=csv,noheader | wc -l
START=$(date +%s)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29518 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench15_n4.json 2> gpurun_out/bench15_n4.err; echo bench4=$? elapsed=$(( $(date +%s) - START ))s
grep -v "^\*\|OMP\|^$" gpurun_out/bench15_n4.err | tail -5
START=$(date +%s)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29519 bench.py --impl reference --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench15_ref4.json 2> gpurun_out/bench15_ref4.err; echo ref4=$? elapsed=$(( $(date +%s) - START ))s
cat gpurun_out/bench15_ref4.json
