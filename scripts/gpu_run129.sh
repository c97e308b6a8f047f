# regression after the codec one-pass paths and the single-stripe pipeline entry
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest129.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest129.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/codec_probe.py 2>&1 | tail -3
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
timeout 900 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "$J"
