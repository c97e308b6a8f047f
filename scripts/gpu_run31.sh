# PIPE input phases (K-split): parity + cfg5 / cfg5d sweeps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -x -k "input_phases" > gpurun_out/pytest31.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest31.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], c["phases"], {k:c["slp"][k] for k in ("xor_count","group_xor","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg5 cfg5d; do
for cfg in "--threads 256 --phases 2" "--threads 128 --phases 1" "--threads 256 --phases 3" "--threads 192 --phases 2" "--threads 128 --phases 2"; do
  echo "== $w $cfg"; timeout 600 python bench.py --workload $w --kernel pipe --stages 2 $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep31.err | python -c "$J"
done; done
