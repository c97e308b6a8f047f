cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 100 --warmup 5"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], {k:d["config"]["slp"][k] for k in ("regs","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg2 pdec; do for cfg in "--threads 256 --lanes 1" "--threads 128 --lanes 2" "--threads 64 --lanes 2" "--threads 128 --lanes 4" "--threads 64 --lanes 4"; do
  echo "== $w pipe $cfg"; $B --workload $w --kernel pipe $cfg 2>/dev/null | python -c "$J"
done; done
for cfg in "--threads 128 --lanes 1" "--threads 64 --lanes 2" "--threads 32 --lanes 4" "--threads 96 --lanes 1"; do
  echo "== cfg5 pipe $cfg"; timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 --warmup 3 --workload cfg5 --kernel pipe $cfg 2>/dev/null | python -c "$J"
done
