# M^-1 fused kernels: reuse 40 / 64 / 96 at 20 per module (cfg3 --kernel multi, xdec at N=1), twice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs"), m.get("modules"), d["clocks"]["sm_mhz"])'
for r in 1 2; do for R in 40 64 96; do
  echo "== cfg3 multi reuse=$R"; timeout 600 python bench.py --workload cfg3 --kernel multi --threads 256 --per-module 20 --reuse $R --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s109.err | python -c "$J"
  echo "== xdec reuse=$R"; timeout 600 python bench.py --workload xdec --reuse $R --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s109.err | python -c "$J"
done; done
