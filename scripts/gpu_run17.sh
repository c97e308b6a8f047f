# fused multi-program decode kernels: parity, then cfg3 sweep (per_module, threads) vs grouped
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "multi_program" > gpurun_out/pytest17.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest17.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], c["stages"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"], d["compile_s"])'
for cfg in "--kernel multi --threads 256 --per-module 64" "--kernel multi --threads 256 --per-module 128" "--kernel multi --threads 256 --per-module 16" "--kernel multi --threads 128 --per-module 64" "--kernel multi --threads 256 --stages 2 --lanes 1 --per-module 700" "--kernel grouped --threads 64"; do
  echo "== cfg3 $cfg"; timeout 900 python bench.py --workload cfg3 --graph 0 $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep17.err | python -c "$J"
done
tail -3 gpurun_out/sweep17.err
