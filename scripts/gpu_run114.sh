# cfg5 (RS(20,4) encode, power-capped) launch sweep with the reuse window: words per thread, phases, window
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c.get("slp") or {}; k=d["clocks"]; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), s.get("spill_bytes_pipe"), k["sm_mhz"], k["power_w"])'
for k in "--threads 256 --phases 2 --reuse 64" "--threads 256 --phases 2 --reuse 32" "--threads 256 --phases 2 --reuse 128" "--threads 128 --lanes 2 --phases 2 --reuse 16" "--threads 128 --lanes 2 --phases 3 --reuse 32" "--threads 128 --lanes 2 --phases 4 --reuse 32" "--threads 256 --phases 3 --reuse 64" "--threads 256 --phases 4 --reuse 64 --stages 3"; do
  echo "== cfg5 $k"; timeout 600 python bench.py --workload cfg5 --kernel pipe $k --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done
