# round 2: the lane-parallel interpreter (interp_lanes.cu, the default XSLP_INTERP_LANES) and the
# pair-pipelined one (--interp pairs): parity + sweep.  CFGS entries: workload_interp_threads_stages_lanes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -n "$NOTEST" ] || { timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "interp or heterogeneous or random_programs or greedy or graph" > gpurun_out/r02l_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02l_pytest.log; }
for cfg in ${CFGS:-cfg2_lanes_512_2_1 pdec_lanes_512_2_1 cfg3_lanes_512_2_1 cfg2_pairs_256_2_1 pdec_pairs_128_2_2 cfg3_pairs_256_2_1}; do
  set -- $(echo $cfg | tr _ " ")
  timeout 300 python bench.py --workload $1 --kernel interp --interp $2 --threads $3 --stages $4 --lanes $5 \
    --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02l_$cfg.json 2> gpurun_out/r02l_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02l_$cfg.json').readline()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel'])" 2>&1 | tail -1)"
done
