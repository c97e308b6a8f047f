cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], c["phases"], c.get("per_module"), c.get("multi"), d["clocks"]["sm_mhz"])'
for cfg in "--threads 128 --lanes 2 --per-module 8" "--threads 128 --lanes 2 --per-module 4" "--threads 128 --lanes 2 --phases 4 --per-module 8"; do
  echo "== cfg5h $cfg"; timeout 1500 python bench.py --workload cfg5h $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s68.err | python -c "$J"
done
for cfg in "--threads 128 --lanes 2 --per-module 20"; do
  echo "== cfg3 $cfg"; timeout 1500 python bench.py --workload cfg3 $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s68.err | python -c "$J"
done
