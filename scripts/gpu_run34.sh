cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -m gpu -k "input_phases or grouped_pipe_with_phases" > gpurun_out/pytest34.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest34.log
