cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --workload cg --steps 3 --warmup 3 --quick"
timeout 600 $CMD > gpurun_out/plain19.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches19_cg.csv $CMD > gpurun_out/ncu_l19.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"spmv|dkf_" -s 12 -c 5 -o gpurun_out/prof_cg19 $CMD > gpurun_out/ncu_full19.log 2>&1; echo ncu2=$?
