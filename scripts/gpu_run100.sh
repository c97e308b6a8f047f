# seeded fuzz of program shapes x launch knobs against the oracle
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -rs -k "random_programs or random_heterogeneous" 2>&1 | tail -25
