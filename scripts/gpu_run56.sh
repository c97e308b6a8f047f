# pipelined interpreter on by default: full GPU suite + interpreter throughput
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest56.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest56.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], d["clocks"]["sm_mhz"], d["gpu_launches"])'
for w in cfg2 pdec cfg3; do for t in 128 256; do
  echo "== $w interp T=$t"; timeout 900 python bench.py --workload $w --kernel interp --threads $t --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep56.err | python -c "$J"
done; done
