# cfg5h with reuse 16: per-module / stages / phases re-sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs"), m.get("modules"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for k in "--per-module 16" "--per-module 8" "--per-module 32" "--per-module 16 --stages 2" "--per-module 16 --phases 4" "--per-module 16 --phases 8" "--per-module 16 --reuse 12" "--per-module 16 --reuse 20" "--per-module 16 --threads 128 --phases 3 --stages 2"; do
  echo "== cfg5h $k"; timeout 600 python bench.py --workload cfg5h $k --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s96.err | python -c "$J"
done
