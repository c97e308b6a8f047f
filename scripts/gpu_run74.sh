cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(c["kernel"], d["steps"], d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for k in "--kernel syndrome --threads 256 --per-module 32" "--kernel multi --threads 256 --per-module 20"; do
  timeout 900 python bench.py --workload cfg3 $k --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>>gpurun_out/s74.err | python -c "$J"
done; done
for k in "--kernel syndrome --threads 128 --per-module 16" "--kernel multi --threads 256 --per-module 8"; do
  timeout 900 python bench.py --workload cfg5h $k --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>>gpurun_out/s74.err | python -c "$J"
done
