# A/B: reuse off vs auto on the workloads that did not gain (cfg2b byte layout, xdec1 LDG), twice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for r in 1 2; do for w in cfg2b xdec1 pdec; do for R in -1 0; do
  echo "== $w reuse=$R"
  timeout 900 python bench.py --workload $w --reuse $R --steps 50 --no-cpu-baseline --no-e2e 2>>gpurun_out/s92.err | python -c "$J"
done; done; done
