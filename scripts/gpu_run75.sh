# full regression with the syndrome defaults: GPU tests, smoke, default bench, cfg3/cfg5h default lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest75.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest75.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench75_default.json 2>gpurun_out/s75.err; echo "bench rc=$?"; cat gpurun_out/bench75_default.json
for w in cfg3 cfg5h; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench75_$w.json 2>>gpurun_out/s75.err; echo "$w rc=$?"; cut -c1-400 gpurun_out/bench75_$w.json
done
