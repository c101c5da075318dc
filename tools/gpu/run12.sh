cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "" "DK_JIT_CS=1" "DK_JIT_UNROLL=4" "DK_JIT_UNROLL=4 DK_JIT_CS=1" "DK_JIT_MINB=2 DK_JIT_UNROLL=4" "DK_JIT_MINB=6" "DK_JIT_UNROLL=1"; do
  for wl in bs stencil cg; do
    R=$(env $cfg timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])")
    echo "cfg=[$cfg] $wl $R"
  done
done
