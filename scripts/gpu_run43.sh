cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "peer" > gpurun_out/pytest43.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest43.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], d["clocks"]["sm_mhz"], d["gpu_launches"])'
echo "== xdec"; timeout 900 python bench.py --workload xdec --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/xdec43.err | python -c "$J"; tail -2 gpurun_out/xdec43.err
