# syndrome-form decode: how much do the number of distinct patterns / modules cost?
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c.get("patterns"), c["multi"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg5h cfg3; do
for a in "--distinct 1" "--distinct 4" "--distinct 16" "--distinct 64" "--distinct 256" ""; do
for t in 128 256; do
  echo "== $w $a T=$t"
  timeout 600 python bench.py --workload $w --kernel syndrome --threads $t --per-module 16 $a --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s77.err | python -c "$J"
done; done; done
