# speed of light for cfg5's traffic (RS(20,4), 2 input phases): RS program vs minimum compute
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do timeout 600 python scripts/sol_probe.py --rs20 2>>gpurun_out/s89.err | tee -a gpurun_out/sol89.jsonl; done
