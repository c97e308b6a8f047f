cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "cuda_graph or single_stripe" 2>&1 | tail -2
