cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload cfg3 > gpurun_out/bench73_cfg3.json 2> gpurun_out/b73.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --workload cfg5h > gpurun_out/bench73_cfg5h.json 2>> gpurun_out/b73.err; echo "cfg5h rc=$?"
python -c "
import json
for f in ('cfg3','cfg5h'):
    d=json.load(open('gpurun_out/bench73_%s.json'%f)); print(f, d['value'], d['roofline']['frac'], d['config']['kernel'], d['clocks'], d['compile_s'], d['cpu_baseline']['value'], d['cpu_baseline']['all_cores']['value'])
"
