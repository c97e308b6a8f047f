# cfg2 A/B: PIPE T=256 L=1 vs T=128 L=2 vs T=64 L=4(?), interleaved, 200 steps each, 3 rounds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], {k:c["slp"][k] for k in ("regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["step_ms"])'
for r in 1 2 3; do
for cfg in "--threads 256 --lanes 1" "--threads 128 --lanes 2" "--threads 192 --lanes 1"; do
  echo "== r$r cfg2 $cfg"; timeout 600 python bench.py --workload cfg2 --kernel pipe --stages 2 $cfg --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab28.err | python -c "$J"
done; done
for cfg in "--threads 256 --lanes 1" "--threads 128 --lanes 2"; do
  echo "== pdec $cfg"; timeout 600 python bench.py --workload pdec --kernel pipe --stages 2 $cfg --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab28.err | python -c "$J"
done
