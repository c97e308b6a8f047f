# M^-1 fused multi-program kernels after the reuse window: per-module x reuse (cfg3 --kernel multi, xdec)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs"), m.get("modules"), d["clocks"]["sm_mhz"])'
for pm in 8 12 20 32; do for R in 16 40; do
  echo "== cfg3 multi pm=$pm reuse=$R"; timeout 600 python bench.py --workload cfg3 --kernel multi --threads 256 --per-module $pm --reuse $R --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s108.err | python -c "$J"
done; done
