cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
XSLP_INTERP_PIPE=1 timeout 1200 python -m pytest tests/test_gpu.py -q -k "interp or lifetime" > gpurun_out/pytest53.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest53.log | head
