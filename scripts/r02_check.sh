# round 2: full GPU test suite + the bench lines touched by this round's changes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
echo "host: $(nproc) cores, $(free -g | awk '/Mem/{print $2}') GiB RAM"
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc=$?"; tail -22 gpurun_out/r02c_pytest.log
for w in ${WLS:-cfg2 cfg5 cfg5d cfg3}; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02c_$w.json 2> gpurun_out/r02c_$w.err
  echo "$w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02c_$w.json').readline()); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['gpu_launches'], (d.get('cpu_baseline') or {}).get('value'), ((d.get('cpu_baseline') or {}).get('one_core') or {}).get('value'), (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"
done
