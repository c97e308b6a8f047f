# byte-layout PIPE launch sweep (cfg2b), twice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c.get("slp") or {}; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), s.get("spill_bytes_pipe"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for k in "--threads 256 --stages 2" "--threads 128 --stages 2" "--threads 128 --stages 3" "--threads 256 --stages 3" "--threads 192 --stages 2" "--threads 64 --stages 4"; do
  echo "== cfg2b $k"; timeout 600 python bench.py --workload cfg2b --kernel pipe $k --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s106.err | python -c "$J"
done; done
