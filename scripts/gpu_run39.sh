# byte layout through the TMA pipeline: parity + throughput vs LDG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -k "byte_layout" > gpurun_out/pytest39.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest39.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], c["stages"], {k:c["slp"][k] for k in ("regs","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for cfg in "--kernel pipe --threads 128 --stages 2" "--kernel pipe --threads 256 --stages 2" "--kernel pipe --threads 128 --stages 3" "--kernel pipe --threads 64 --stages 4" "--kernel straight --threads 128"; do
  echo "== cfg2b $cfg"; timeout 600 python bench.py --workload cfg2b $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep39.err | python -c "$J"
done
