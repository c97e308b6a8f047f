# RS(20,4) PIPE with 2 lanes per thread (LDS.64: half the shared-memory load instructions)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], c["stages"], {k:c["slp"][k] for k in ("regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg5 cfg5d; do
for cfg in "--threads 64 --lanes 2 --stages 2" "--threads 128 --lanes 1 --stages 2" "--threads 96 --lanes 1 --stages 2"; do
  echo "== $w $cfg"; timeout 600 python bench.py --workload $w --kernel pipe $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep24.err | python -c "$J"
done; done
for cfg in "--threads 128 --lanes 2 --stages 2" "--threads 64 --lanes 2 --stages 3" "--threads 256 --lanes 1 --stages 2"; do
  echo "== cfg2 $cfg"; timeout 600 python bench.py --workload cfg2 --kernel pipe $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep24.err | python -c "$J"
done
