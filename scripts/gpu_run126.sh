cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_codec.py -x -q 2>&1 | tail -2
