# experiment: one CTA per SM per module launch (two modules share each SM on the two streams)
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'
for r in 1 2; do for w in cfg5h cfg3; do for c in 0 1; do
  echo "== $w cap=$c"; XSLP_MULTI_CTAS_PER_SM=$c timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "$J"
done; done; done
