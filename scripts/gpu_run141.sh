# P_dec: launch variants with 2 input phases x 3 stages (30 steps, twice)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c["slp"]; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), d["clocks"]["sm_mhz"])'
for r in 1 2; do
for k in "" "--threads 256 --lanes 1 --phases 2 --stages 3" "--phases 2 --stages 3 --reuse 32" "--reuse 32"; do
  echo "== pdec $k"; timeout 600 python bench.py --workload pdec $k --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done
