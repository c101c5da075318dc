cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_session.py -q -x > gpurun_out/pytest_gpu8.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu8.log
CMD2="python bench.py --workload stencil --steps 5 --warmup 3 --no-extra"
timeout 600 $CMD2 > gpurun_out/bench8_st.json 2> gpurun_out/bench8_st.err; echo bench=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dkf_ -s 6 -c 2 -o gpurun_out/prof_st8 $CMD2 > gpurun_out/ncu_full8.log 2>&1; echo ncu=$?
