# regression with the constant reuse window on by default: all GPU tests, smoke, every workload's line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest91.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest91.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
timeout 900 python bench.py > gpurun_out/bench91_default.json 2>>gpurun_out/s91.err; echo "default rc=$?"; python -c "$J" < gpurun_out/bench91_default.json
for w in pdec cfg3 cfg5 cfg5d cfg5h cfg2b xdec1; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench91_$w.json 2>>gpurun_out/s91.err; echo "$w rc=$?"; python -c "$J" < gpurun_out/bench91_$w.json
done
