# more stages with smaller input phases for the other lines (30 steps, twice)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or c.get("slp") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs") or m.get("regs_pipe"), d["clocks"]["sm_mhz"])'
for r in 1 2; do
for k in "" "--phases 4 --stages 3" "--phases 4 --stages 4" "--phases 7 --stages 3"; do
  echo "== cfg3 $k"; timeout 600 python bench.py --workload cfg3 $k --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done
for k in "" "--phases 4 --stages 3" "--phases 4 --stages 4"; do
  echo "== cfg5 $k"; timeout 600 python bench.py --workload cfg5 $k --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done
