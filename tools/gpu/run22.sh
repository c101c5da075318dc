cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "DK_TMA_L2=256" "DK_TMA_L2=128" "DK_TMA_L2=0" "DK_TMA_L2=64"; do
    R=$(env $cfg timeout 600 python bench.py --workload stencil --steps 20 --warmup 3 --quick 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['hbm_gbs_step'])")
    echo "cfg=[$cfg] stencil $R"
done
done
CMD2="python bench.py --workload stencil --steps 2 --warmup 3 --quick"
DK_TMA_L2=0 timeout 600 $CMD2 > /dev/null 2>&1 && DK_TMA_L2=0 timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dkf_ -s 6 -c 2 --csv $CMD2 2>/dev/null | grep -E "dram|duration" | tail -6
