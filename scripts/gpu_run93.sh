# ncu of the default line's kernel with the constant reuse window (launch list + --set full),
# and of cfg5 (RS(20,4), 2 phases) with it
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain93.json 2>gpurun_out/s93.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches93.csv $C > /dev/null 2>>gpurun_out/s93.err; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof93_cfg2 $C > /dev/null 2>>gpurun_out/s93.err; echo "full rc=$?"
C5="python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 8 -c 1 -o gpurun_out/prof93_cfg5 $C5 > /dev/null 2>>gpurun_out/s93.err; echo "full5 rc=$?"
