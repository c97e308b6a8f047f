# cfg5h syndrome-form launch sweep (1 distinct pattern and all patterns)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["multi"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for a in "--distinct 1" ""; do
for k in "--threads 128 --phases 2" "--threads 128 --phases 3 --stages 3" "--threads 128 --phases 4 --stages 3" "--threads 256 --phases 4" "--threads 256 --phases 6" "--threads 256 --phases 3 --stages 3" "--threads 64 --phases 3 --stages 3" "--threads 128 --phases 6 --stages 4"; do
  echo "== cfg5h $a $k"
  timeout 600 python bench.py --workload cfg5h --kernel syndrome --per-module 16 $a $k --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s78.err | python -c "$J"
done; done
