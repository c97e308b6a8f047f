# confirm the new syndrome module sizes: full-size parity in the bench config, 100-step lines twice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "syndrome_full_size" 2>&1 | tail -1
for r in 1 2; do for w in cfg3 cfg5h; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench98_${w}_$r.json 2>>gpurun_out/s98.err; echo "$w rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench98_${w}_$r.json')); print(d['value'], d['roofline']['frac'], d['clocks'], d['config']['multi'])"
done; done
