cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu51.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu51.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench51.json 2> gpurun_out/bench51.err; echo bench=$?
CMD2="python bench.py --workload stencil --steps 5 --warmup 3 --no-extra"
timeout 600 $CMD2 > gpurun_out/bench51_st.json 2> gpurun_out/bench51_st.err; echo bench_st=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dkf_ -s 6 -c 2 -o gpurun_out/prof_st51 $CMD2 > gpurun_out/ncu_full51.log 2>&1; echo ncu=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches51_st.csv $CMD2 > gpurun_out/ncu_launch51.log 2>&1; echo ncu_l=$?
