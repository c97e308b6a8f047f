# ncu captures: cfg5 PIPE T=128 (groups 1 and 2) and the cfg3 grouped launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof_cfg5_g1 \
   $B --workload cfg5 --kernel pipe --threads 128 --groups 1 > gpurun_out/ncu16a.log 2>&1; echo "a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof_cfg5_g2 \
   $B --workload cfg5 --kernel pipe --threads 128 --groups 2 > gpurun_out/ncu16b.log 2>&1; echo "b rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes.sum.per_second --clock-control none -k regex:xslp_sl --csv --log-file gpurun_out/launches_cfg3.csv \
   python bench.py --workload cfg3 --graph 0 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu16c.log 2>&1; echo "c rc=$?"
