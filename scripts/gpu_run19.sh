# ncu: multi kernel launches at per_module 64 and 128 (stall reasons: icache = no_instruction)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --workload cfg3 --graph 0 --kernel multi --threads 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 14 -c 1 -o gpurun_out/prof_multi64 $B --per-module 64 > gpurun_out/ncu19a.log 2>&1; echo "a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 8 -c 1 -o gpurun_out/prof_multi128 $B --per-module 128 > gpurun_out/ncu19b.log 2>&1; echo "b rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes.sum.per_second,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio --clock-control none -k regex:xslp_sl_multi --csv --log-file gpurun_out/launches_multi64.csv $B --per-module 64 > gpurun_out/ncu19c.log 2>&1; echo "c rc=$?"
