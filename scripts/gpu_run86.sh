# speed of light for the cfg2 traffic mix: RS(10,4) program vs minimum-compute program, same PIPE launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do timeout 600 python scripts/sol_probe.py 2>>gpurun_out/s86.err | tee -a gpurun_out/sol86.jsonl; done
