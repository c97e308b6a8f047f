# full regression: all GPU tests (incl. fuzz), smoke, default line, every workload's line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest104.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest104.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], (d.get("e2e") or {}).get("value"))'
timeout 900 python bench.py > gpurun_out/bench104_default.json 2>>gpurun_out/s104.err; echo "default rc=$?"; python -c "$J" < gpurun_out/bench104_default.json
for w in pdec cfg3 cfg5 cfg5d cfg5h cfg2b cfg2t xdec xdec1; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench104_$w.json 2>>gpurun_out/s104.err; echo "$w rc=$?"; python -c "$J" < gpurun_out/bench104_$w.json
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench104_reference.json 2>>gpurun_out/s104.err; echo "reference rc=$?"; cut -c1-200 gpurun_out/bench104_reference.json
