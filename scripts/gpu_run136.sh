# 100-step A/B: cfg2 / pdec default launch vs 2 input phases x 3 stages (alternating, twice)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do for w in cfg2 pdec; do for k in "" "--phases 2 --stages 3"; do
  echo "== $w $k"; timeout 600 python bench.py --workload $w $k --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done; done
