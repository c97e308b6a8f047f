# cfg3 default line (multi) + per_module sweep + multi with 2 stages at T=224
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], c["stages"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"], d["compile_s"])'
for cfg in "--per-module 48" "--per-module 80" "--per-module 56" "--per-module 64 --threads 224"; do
  echo "== cfg3 multi $cfg"; timeout 900 python bench.py --workload cfg3 $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep20.err | python -c "$J"
done
timeout 900 python bench.py --workload cfg3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
cat gpurun_out/bench_cfg3.json
