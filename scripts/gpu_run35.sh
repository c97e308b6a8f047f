# experiment: multi kernel tile order contiguous vs strided
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c.get("per_module"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for pm in 56 28; do
  echo "== contiguous pm=$pm"; timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep35.err | python -c "$J"
  echo "== strided pm=$pm"; XSLP_MULTI_STRIDED=1 timeout 900 python bench.py --workload cfg3 --per-module $pm --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep35.err | python -c "$J"
done; done
XSLP_MULTI_STRIDED=1 timeout 900 python -m pytest tests/test_gpu.py -q -k multi_program > gpurun_out/pytest35.log 2>&1; echo "pytest strided rc=$?"; tail -1 gpurun_out/pytest35.log
