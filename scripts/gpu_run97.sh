# cfg5h per-module sweep with reuse 16 (twice), and cfg3 per-module with reuse 40
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs"), m.get("modules"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for pm in 4 6 8 10 12; do
  echo "== cfg5h pm=$pm"; timeout 600 python bench.py --workload cfg5h --per-module $pm --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s97.err | python -c "$J"
done
for pm in 8 16 32 64; do
  echo "== cfg3 pm=$pm"; timeout 600 python bench.py --workload cfg3 --per-module $pm --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s97.err | python -c "$J"
done; done
