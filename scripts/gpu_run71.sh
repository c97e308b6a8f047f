# syndrome-form heterogeneous decode: cfg3 and cfg5h
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["threads"], c["phases"], c.get("per_module"), c.get("multi"), d["compile_s"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg3 cfg5h; do for cfg in "--threads 256 --per-module 64" "--threads 256 --per-module 256" "--threads 128 --per-module 64" "--threads 256 --per-module 64 --phases 1"; do
  echo "== $w syndrome $cfg"; timeout 1500 python bench.py --workload $w --kernel syndrome $cfg --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s71.err | python -c "$J"
done; done
tail -2 gpurun_out/s71.err
