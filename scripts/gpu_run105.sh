# xdec1 at N=1 through the TMA pipeline (all blocks local); peer tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "peer" 2>&1 | tail -1
timeout 900 python bench.py --workload xdec1 --no-cpu-baseline --no-e2e > gpurun_out/bench105_xdec1.json 2>gpurun_out/s105.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench105_xdec1.json')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks'])"
