# final state: all GPU tests, smoke, the default line five times, the default line with cpu_baseline + e2e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest139.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest139.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
: > gpurun_out/repeat139.jsonl
for i in 1 2 3 4 5; do timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null >> gpurun_out/repeat139.jsonl; done
python -c "
import json
for l in open('gpurun_out/repeat139.jsonl'):
    d=json.loads(l); c=d['clocks']; print(d['value'], d['roofline']['frac'], d['step_ms'], c['sm_mhz'], c['reasons'])
"
timeout 900 python bench.py > gpurun_out/bench139_default.json 2>gpurun_out/s139.err; echo "default rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench139_default.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
