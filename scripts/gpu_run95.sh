# per-workload reuse windows: the affected parity tests, smoke, default + cfg3 lines (100 steps, twice)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cfg2_full_size or syndrome_full_size or const_reuse" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("e2e",{}).get("value"))'
timeout 900 python bench.py > gpurun_out/bench95_default.json 2>>gpurun_out/s95.err; echo "default rc=$?"; python -c "$J" < gpurun_out/bench95_default.json
for r in 1 2; do
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --no-e2e > gpurun_out/bench95_cfg3_$r.json 2>>gpurun_out/s95.err; echo "cfg3 rc=$?"; python -c "$J" < gpurun_out/bench95_cfg3_$r.json
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench95_cfg2_$r.json 2>>gpurun_out/s95.err; echo "cfg2 rc=$?"; python -c "$J" < gpurun_out/bench95_cfg2_$r.json
done
