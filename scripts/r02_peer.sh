# round 2: cross-GPU decode (NEXT #4) -- IPC peer tables through the LDG kernel and the opt-in
# TMA-staged kernels; the two-device tests run when the box has >= 2 GPUs (they skip otherwise)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu.py -q -k "peer" -rs > gpurun_out/r02p_pytest.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/r02p_pytest.log
