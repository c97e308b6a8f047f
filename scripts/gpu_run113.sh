# power next to clocks for the default line and the RS(20,4) lines
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"])'
for w in cfg2 cfg5 cfg5h; do echo "== $w"; timeout 600 python bench.py --workload $w --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"; done
