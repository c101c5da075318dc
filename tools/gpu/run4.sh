cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench=$?
CMD="python bench.py --steps 3 --warmup 3 --no-extra"
timeout 600 $CMD > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv $CMD > gpurun_out/ncu_launch4.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dkf_ -s 3 -c 1 -o gpurun_out/prof_bs4 $CMD > gpurun_out/ncu_full4.log 2>&1; echo ncu2=$?
CMD2="python bench.py --workload stencil --steps 2 --warmup 3 --no-extra"
timeout 600 $CMD2 > gpurun_out/plain4s.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dkf_ -s 6 -c 2 -o gpurun_out/prof_st4 $CMD2 > gpurun_out/ncu_full4s.log 2>&1; echo ncu3=$?
