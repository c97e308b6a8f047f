# full GPU suite + smoke + default bench line + cfg3 line (regression check after session-2 changes)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke23.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke23.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest23.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest23.log
timeout 600 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err; echo "bench rc=$?"; cat gpurun_out/bench23.json
timeout 900 python bench.py --workload cfg3 > gpurun_out/bench23_cfg3.json 2> gpurun_out/bench23_cfg3.err; echo "cfg3 rc=$?"; cut -c1-400 gpurun_out/bench23_cfg3.json
