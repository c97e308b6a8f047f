# RS(10,4) with input phases: more consumer warps / more stages per SM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["lane_words"], c["stages"], c["phases"], {k:c["slp"][k] for k in ("group_xor","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for cfg in "--threads 128 --lanes 2 --stages 2 --phases 1" "--threads 256 --lanes 2 --stages 2 --phases 2" "--threads 256 --lanes 1 --stages 4 --phases 2" "--threads 256 --lanes 1 --stages 3 --phases 2" "--threads 128 --lanes 2 --stages 4 --phases 2" "--threads 512 --lanes 1 --stages 2 --phases 2"; do
  echo "== cfg2 $cfg"; timeout 600 python bench.py --workload cfg2 --kernel pipe $cfg --steps 100 --warmup 10 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep57.err | python -c "$J"
done
