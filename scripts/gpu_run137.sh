# new default launch (2 input phases x 3 stages): parity in that config, smoke, the default line,
# ncu launch list + full capture of its kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "cfg2_full_size or bench_contract or readme or input_phases or const_reuse" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench137_default.json 2>gpurun_out/s137.err; echo "default rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench137_default.json')); print(d['value'], d['roofline'], d['e2e']['value'], d['clocks'])"
C="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches137.csv $C > /dev/null 2>>gpurun_out/s137.err; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof137_cfg2 $C > /dev/null 2>>gpurun_out/s137.err; echo "full rc=$?"
