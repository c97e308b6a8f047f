cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "multi_program or peer" > gpurun_out/pytest61.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest61.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for r in 1 2; do timeout 900 python bench.py --workload cfg3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s61.err | python -c "$J"; done
