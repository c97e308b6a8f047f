# multi kernel with two internal streams: parity (+graph) and cfg3 line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "multi_program or graph" > gpurun_out/pytest22.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest22.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c.get("per_module"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"])'
for pm in 56 64 40; do
  echo "== cfg3 multi pm=$pm"; timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep22.err | python -c "$J"
done
