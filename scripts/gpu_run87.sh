# speed of light for the cfg2 traffic mix: RS(10,4) program vs minimum-compute program, same PIPE launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/sol_probe.py --mix 2>>gpurun_out/s87.err | tee -a gpurun_out/sol87.jsonl
