# new full-size tests; cfg2t line with the ALU roofline; cfg5h / cfg3 default lines (100 steps)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "syndrome_full_size or gf_table" 2>&1 | tail -2
for w in cfg2t cfg5h cfg3; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench84_$w.json 2>>gpurun_out/s84.err; echo "$w rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench84_$w.json')); print(d['value'], d['roofline'], d['clocks'])"
done
