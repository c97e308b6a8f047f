# P_dec on its new launch (T=256, 2 phases x 3 stages): full-size parity and the 100-step line
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "pdec" 2>&1 | tail -1
timeout 600 python bench.py --workload pdec --no-cpu-baseline --no-e2e > gpurun_out/bench143_pdec.json 2>/dev/null; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench143_pdec.json')); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['config']['threads'], d['config']['phases'], d['config']['stages'])"
