# multi kernel with 2 words per thread
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "multi_program" > gpurun_out/pytest30.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest30.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], c.get("per_module"), c.get("multi"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for cfg in "--threads 128 --lanes 2 --per-module 56" "--threads 128 --lanes 2 --per-module 40" "--threads 128 --lanes 2 --per-module 28" "--threads 256 --lanes 1 --per-module 56"; do
  echo "== cfg3 $cfg"; timeout 900 python bench.py --workload cfg3 $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep30.err | python -c "$J"
done
