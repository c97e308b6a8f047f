cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["kernel"], c["parallelism"][:60], d["gpu_launches"])'
for w in xdec1 xdec; do
  echo "== $w staged"; timeout 900 python bench.py --workload $w --xmode staged --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/xs46_$w.err | python -c "$J"; tail -1 gpurun_out/xs46_$w.err
done
