cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu.py -q -rs -k "random_programs" 2>&1 | tail -4
