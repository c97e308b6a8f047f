# DRAM bytes per launch (ncu launch lists) for the workloads without a traffic entry yet
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in pdec cfg5d xdec1 xdec cfg2b; do
  C="python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  $C > gpurun_out/plain102_$w.json 2>>gpurun_out/s102.err; echo "$w plain rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches102_$w.csv $C > /dev/null 2>>gpurun_out/s102.err; echo "$w ncu rc=$?"
done
