cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "" "DK_JIT_MINB=6" "DK_JIT_MINB=4" "DK_JIT_MINB=8" ; do
  for wl in bs; do
    R=$(env $cfg timeout 600 python bench.py --workload $wl --steps 30 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])")
    echo "cfg=[$cfg] $wl $R"
  done
done
for cfg in "" "DK_JIT_MINB=2" "DK_JIT_MINB=3" "DK_JIT_NO_K3=1"; do
    R=$(env $cfg timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['kernel'])")
    echo "cfg=[$cfg] stencil $R"
done
done
