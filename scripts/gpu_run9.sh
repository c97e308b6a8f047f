# round-1 call 9: graph capture tests + compute-sanitizer memcheck over every kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu9.log



