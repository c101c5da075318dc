cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 4000000 8000000; do
N=$n TAG="n=$n" timeout 300 python tools/gpu/jitprobe.py 2>&1 | tail -2
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
