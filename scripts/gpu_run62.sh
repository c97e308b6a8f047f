cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "multi_program or peer" > gpurun_out/pytest62.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest62.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["config"].get("per_module"), d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["gpu_launches"])'
for pm in 12 20 28 40 56; do timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s62.err | python -c "$J"; done
