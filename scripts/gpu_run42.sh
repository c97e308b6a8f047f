# regression: smoke + full GPU suite + default line + reference arm + cfg3/cfg2b lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke42.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke42.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest42.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest42.log
timeout 600 python bench.py > gpurun_out/bench42.json 2> gpurun_out/bench42.err; echo "bench rc=$?"; cut -c1-250 gpurun_out/bench42.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench42_ref.json 2>> gpurun_out/bench42.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/bench42_ref.json
timeout 900 python bench.py --workload cfg3 > gpurun_out/bench42_cfg3.json 2>> gpurun_out/bench42.err; echo "cfg3 rc=$?"; cut -c1-200 gpurun_out/bench42_cfg3.json
timeout 900 python bench.py --workload cfg2b > gpurun_out/bench42_cfg2b.json 2>> gpurun_out/bench42.err; echo "cfg2b rc=$?"; cut -c1-200 gpurun_out/bench42_cfg2b.json
