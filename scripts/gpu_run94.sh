# finer reuse-window sweep around the defaults (fused kernels: 8-40; single-program: 32-128), twice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c.get("slp") or {}; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe") or m.get("regs"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for W in 8 16 24 32 40; do for w in cfg3 cfg5h; do
  echo "== $w W=$W"; timeout 600 python bench.py --workload $w --reuse $W --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s94.err | python -c "$J"
done; done
for W in 32 64 96 128; do for w in cfg2 cfg5d; do
  echo "== $w W=$W"; timeout 600 python bench.py --workload $w --reuse $W --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s94.err | python -c "$J"
done; done; done
