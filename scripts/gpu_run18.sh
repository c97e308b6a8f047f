# multi kernel v2 (producer-resolved tile headers): parity + cfg3 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "multi_program" > gpurun_out/pytest18.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest18.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], c["stages"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"], d["compile_s"])'
for cfg in "--threads 256 --per-module 64" "--threads 256 --per-module 128" "--threads 256 --per-module 32" "--threads 128 --per-module 64" "--threads 128 --stages 3 --per-module 64" "--threads 192 --per-module 64"; do
  echo "== cfg3 multi $cfg"; timeout 900 python bench.py --workload cfg3 --graph 0 --kernel multi $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep18.err | python -c "$J"
done
tail -2 gpurun_out/sweep18.err
