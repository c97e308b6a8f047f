# reproducibility: the default line five times back to back (100 steps each), plus pdec and cfg3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/repeat116.jsonl
for i in 1 2 3 4 5; do timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null >> gpurun_out/repeat116.jsonl; done
for w in pdec cfg3; do for i in 1 2 3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null >> gpurun_out/repeat116.jsonl; done; done
python -c "
import json
for l in open('gpurun_out/repeat116.jsonl'):
    d=json.loads(l); c=d['clocks']; print(d['config']['workload'][:5], d['value'], d['roofline']['frac'], d['step_ms']['min'], d['step_ms']['max'], c['sm_mhz'], c['power_w'], c['reasons'])
"
