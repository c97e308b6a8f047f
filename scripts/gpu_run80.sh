# cfg5h syndrome-form: T=256 with more input phases, per-module sweep (two passes for noise)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["multi"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do
for k in "--phases 6 --per-module 16" "--phases 6 --per-module 8" "--phases 6 --per-module 32" "--phases 8 --per-module 16" "--phases 12 --per-module 16" "--phases 6 --per-module 16 --stages 3" "--phases 8 --per-module 16 --stages 3"; do
  echo "== cfg5h T=256 $k"
  timeout 600 python bench.py --workload cfg5h --kernel syndrome --threads 256 $k --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s80.err | python -c "$J"
done; done
