# single-stripe pipeline entry: parity, the single-stripe / codec tests, codec throughput
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "single_stripe or codec or edge or readme or smoke or one" 2>&1 | tail -2
timeout 600 python scripts/codec_probe.py 2>&1 | tail -3
