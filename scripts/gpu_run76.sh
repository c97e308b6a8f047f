# ncu --set full of the syndrome-form decode kernels (cfg5h, cfg3) + launch lists
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg5h cfg3; do
C="python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$C > gpurun_out/ncu76_${w}_plain.json 2>gpurun_out/s76.err; echo "$w plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches76_$w.csv $C > /dev/null 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 30 -c 1 -o gpurun_out/prof76_$w $C > gpurun_out/ncu76_$w.log 2>&1; echo "full rc=$?"
done
