# pipelined interpreter throughput, T = 128 / 256 (A/B against the previous consumer loop: run on both builds)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], d["clocks"]["sm_mhz"])'
for r in 1 2; do for w in cfg2 pdec; do for t in 128 256; do
  echo "== $w interp T=$t"; timeout 900 python bench.py --workload $w --kernel interp --threads $t --lanes 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done; done
