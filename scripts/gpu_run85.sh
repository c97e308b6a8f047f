# per-step DRAM traffic of the syndrome-form decode (cfg3, cfg5h defaults): ncu launch list with
# dram bytes for every launch of a 1-step run; full capture of one cfg5h kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg3 cfg5h; do
C="python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain85_$w.json 2>>gpurun_out/s85.err; echo "$w plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches85_$w.csv $C > /dev/null 2>>gpurun_out/s85.err; echo "launch rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 200 -c 1 -o gpurun_out/prof85_cfg5h python bench.py --workload cfg5h --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>>gpurun_out/s85.err; echo "full rc=$?"
