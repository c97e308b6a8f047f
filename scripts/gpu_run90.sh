# constant register reuse window (XSLP_CONST_REUSE) sweep: fewer shared-memory reads vs registers
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c.get("slp") or {}; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), s.get("spill_bytes_pipe"), c.get("multi"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for W in 0 16 64 256; do
for a in "cfg2" "cfg2 --threads 256 --lanes 1" "pdec" "cfg5 --steps 10" "cfg5d --steps 10" "cfg3" "cfg5h"; do
  echo "== W=$W $a"
  XSLP_CONST_REUSE=$W timeout 600 python bench.py --steps 30 --workload $a --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s90.err | python -c "$J"
done; done
