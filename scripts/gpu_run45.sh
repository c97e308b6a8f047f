# after refactoring the pipeline emitters: full GPU suite + default line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest45.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest45.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench45.json 2> gpurun_out/bench45.err; echo "bench rc=$?"; cut -c1-220 gpurun_out/bench45.json
