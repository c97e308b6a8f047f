cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "graph_capture" > gpurun_out/pytest44.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest44.log
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof_byte_pipe $B --workload cfg2b > gpurun_out/ncu44a.log 2>&1; echo "a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 40 -c 1 -o gpurun_out/prof_multi20 $B --workload cfg3 > gpurun_out/ncu44b.log 2>&1; echo "b rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:xslp_sl_multi --csv --log-file gpurun_out/launches_multi20.csv python bench.py --workload cfg3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu44c.log 2>&1; echo "c rc=$?"
