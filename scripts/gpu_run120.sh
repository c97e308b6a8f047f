# approach (1) kernel with 4 x 16 B per thread (experiment)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "gf_table" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["hbm"]["frac"], d["clocks"]["sm_mhz"])'
for r in 1 2; do timeout 600 python bench.py --workload cfg2t --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"; done
