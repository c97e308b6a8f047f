# cfg5 / cfg5d launch sweep (RS(20,4): 20:4 read:write leaves ~6% to the mix probe's ceiling)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; s=c["slp"]; print(d["value"], d["roofline"]["frac"], s.get("regs_pipe"), s.get("spill_bytes_pipe"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg5 cfg5d; do
for k in "--threads 256 --stages 2 --phases 2" "--threads 256 --stages 3 --phases 2" "--threads 128 --lanes 2 --stages 2 --phases 2" "--threads 128 --lanes 2 --stages 2 --phases 4" "--threads 256 --stages 2 --phases 4" "--threads 256 --stages 4 --phases 4" "--threads 128 --stages 3 --phases 2"; do
  echo "== $w $k"
  timeout 600 python bench.py --workload $w --kernel pipe $k --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s88.err | python -c "$J"
done; done
