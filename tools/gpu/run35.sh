cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/gpu/mixprobe.py 2>&1 | grep add
for v in "TAG=default" "DK_JIT_MINB=4" "DK_JIT_MINB=8" "DK_JIT_UNROLL=4" "DK_JIT_UNROLL=1" "DK_JIT_UNROLL=4 DK_JIT_MINB=4" "DK_JIT_CS=1"; do
env TAG="$v" $v timeout 300 python tools/gpu/jitprobe.py 2>&1 | tail -2
done
