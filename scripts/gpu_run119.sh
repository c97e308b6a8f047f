# sustained runs with the current defaults (power cap): default line 1000 / 5000 steps, cfg5 100 steps
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["clocks"]; print(d["steps"], d["value"], d["roofline"]["frac"], d["ms_per_step"], c["sm_mhz"], c["power_w"], c["reasons"])'
for s in 1000 5000; do echo "== cfg2 steps=$s"; timeout 900 python bench.py --steps $s --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"; done
echo "== cfg5 steps=100"; timeout 900 python bench.py --workload cfg5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
