cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["phases"], c.get("per_module"), c.get("multi"), d["clocks"]["sm_mhz"])'
for cfg in "--per-module 3" "--per-module 5" "--per-module 8" "--per-module 5 --stages 2 --threads 192"; do
  echo "== cfg5h $cfg"; timeout 1500 python bench.py --workload cfg5h $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s66.err | python -c "$J"
done
echo "== grouped (one PIPE kernel per pattern, phases)"; timeout 1500 python bench.py --workload cfg5h --kernel grouped_pipe --threads 256 --steps 10 --warmup 2 --no-e2e --no-cpu-baseline 2>>gpurun_out/s66.err | python -c "$J"
echo "== interp"; timeout 1500 python bench.py --workload cfg5h --kernel interp --threads 128 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>>gpurun_out/s66.err | python -c "$J"
tail -2 gpurun_out/s66.err
