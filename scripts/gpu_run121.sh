# final-state regression: all GPU tests, smoke, default line (as the driver runs it), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest121.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest121.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench121_default.json 2>gpurun_out/s121.err; echo "default rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench121_default.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/bench121_reference.json 2>>gpurun_out/s121.err; echo "reference rc=$?"; cut -c1-160 gpurun_out/bench121_reference.json
