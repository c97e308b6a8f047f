# P_dec 100-step A/B (alternating, twice)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for r in 1 2; do
for k in "" "--threads 256 --lanes 1 --phases 2 --stages 3" "--phases 2 --stages 3 --reuse 32"; do
  echo "== pdec $k"; timeout 600 python bench.py --workload pdec $k --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done
