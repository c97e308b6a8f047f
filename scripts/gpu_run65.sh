# phased multi-program kernels for wide codes: parity + cfg5h (RS(20,4) per-stripe patterns)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -k "multi_program" > gpurun_out/pytest65.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest65.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["phases"], c.get("per_module"), c.get("patterns"), c.get("multi"), d["compile_s"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for cfg in "--phases 0 --per-module 20" "--phases 1 --threads 128 --per-module 20" "--phases 0 --per-module 10"; do
  echo "== cfg5h $cfg"; timeout 1500 python bench.py --workload cfg5h $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s65.err | python -c "$J"
done
tail -2 gpurun_out/s65.err
