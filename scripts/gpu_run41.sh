cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c.get("per_module"), c.get("multi"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"])'
for pm in 4 8 12 20 56; do
  echo "== cfg3 pm=$pm"; timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep41.err | python -c "$J"
done
