cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "syndrome" > gpurun_out/pytest70.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest70.log
