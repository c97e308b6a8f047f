# CUDA-graph replay of a whole step for the many-launch workloads (cfg5h 98 launches, cfg3 41)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["cuda_graph"], d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do for w in cfg5h cfg3; do for g in 0 1; do
  echo "== $w graph=$g"; timeout 600 python bench.py --workload $w --graph $g --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/s111.err | python -c "$J"
done; done; done
tail -3 gpurun_out/s111.err
