# cfg2 with input phases + more stages now that the reuse window is on (twice, 30 steps)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c["slp"]; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), s.get("spill_bytes_pipe"), d["clocks"]["sm_mhz"])'
for r in 1 2; do
for k in "" "--phases 2 --stages 3" "--phases 2 --stages 4" "--threads 256 --lanes 1 --phases 2 --stages 3" "--threads 256 --lanes 1 --reuse 64"; do
  echo "== cfg2 $k"; timeout 600 python bench.py $k --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done
