# leaner pipelined-interpreter consumer loop (goal pointers in the tile header, mask reset, branch-
# guarded goal store): interpreter parity tests and lines
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "interp or codec or random_programs" 2>&1 | tail -2
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for w in cfg2 pdec cfg3; do echo "== $w interp"; timeout 600 python bench.py --workload $w --kernel interp --threads 128 --graph 0 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"; done
