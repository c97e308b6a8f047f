cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "multi_program" > gpurun_out/pytest38.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest38.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c.get("per_module"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for pm in 56 28 14; do
  echo "== cfg3 PDL pm=$pm"; timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep38.err | python -c "$J"
done
timeout 600 python scripts/multi_probe.py
