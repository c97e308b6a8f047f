cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu.py -m gpu -x -q -k "grid_limit or widest or concurrent or graph" > gpurun_out/pytest_gpu10.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu10.log
