# round-1 call 7: parity suite (full-size cases in bench launch configs) + cfg4 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu7.log
timeout 2400 bash scripts/cfg4_sweep.sh > gpurun_out/cfg4_table.md 2> gpurun_out/cfg4.err
echo "cfg4 rc=$?"; cat gpurun_out/cfg4_table.md
