cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["phases"], c.get("per_module"), c.get("multi"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for cfg in "--threads 128 --per-module 32" "--threads 128 --per-module 16" "--threads 192 --per-module 32" "--threads 128 --per-module 32 --phases 2" "--threads 128 --per-module 32 --phases 4" "--threads 128 --per-module 32 --stages 3"; do
  echo "== cfg5h syndrome $cfg"; timeout 1500 python bench.py --workload cfg5h --kernel syndrome $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s72.err | python -c "$J"
done
for cfg in "--threads 256 --per-module 32" "--threads 256 --per-module 128" "--threads 256 --per-module 64 --phases 3"; do
  echo "== cfg3 syndrome $cfg"; timeout 1500 python bench.py --workload cfg3 --kernel syndrome $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s72.err | python -c "$J"
done
