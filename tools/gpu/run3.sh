cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench=$?
CMD="python bench.py --steps 3 --warmup 3 --no-extra"
timeout 600 $CMD > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $CMD > gpurun_out/ncu_launch3.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dkf_ -s 3 -c 1 -o gpurun_out/prof_bs3 $CMD > gpurun_out/ncu_full3.log 2>&1; echo ncu2=$?
