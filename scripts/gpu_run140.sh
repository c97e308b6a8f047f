# sustained runs of the final default launch under the power cap
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["clocks"]; print(d["steps"], d["value"], d["roofline"]["frac"], d["step_ms"], c["sm_mhz"], c["power_w"], c["reasons"])'
for s in 1000 5000; do timeout 900 python bench.py --steps $s --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"; done
