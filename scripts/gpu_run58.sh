# sustained runs of the default line (power cap behaviour)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["steps"], d["value"], d["roofline"]["frac"], d["clocks"], d["step_ms"])'
for st in 100 1000 5000; do
  echo "== cfg2 steps=$st"; timeout 900 python bench.py --steps $st --warmup 20 --no-e2e --no-cpu-baseline 2>>gpurun_out/sus58.err | python -c "$J"
done
echo "== cfg5 steps=100 (sustained, 2048-stripe chunks)"; timeout 900 python bench.py --workload cfg5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sus58.err | python -c "$J"
