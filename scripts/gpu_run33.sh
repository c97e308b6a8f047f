cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_codec.py -q -m gpu -k "lifetime or every_4_loss" --durations=5 > gpurun_out/pytest33.log 2>&1
echo "pytest rc=$?"; tail -12 gpurun_out/pytest33.log
