# round 2: the TMEM interpreter (interp_tmem.cu, --interp tmem): parity + bench lines.
# CFGS entries: workload_lanes_threads_stages_batch (batch: XSLP_TMEM_BATCH, ops per batch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -n "$NOTEST" ] || { timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "${TK:-tmem}" > gpurun_out/r02t_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02t_pytest.log; }
for cfg in ${CFGS:-cfg2_2_128_2_8 cfg2_2_128_2_4 cfg2_1_256_2_8 pdec_2_128_2_8 cfg3_2_128_2_8}; do
  set -- $(echo $cfg | tr _ " ")
  XSLP_TMEM_BATCH=$5 timeout 300 python bench.py --workload $1 --kernel interp --interp tmem --lanes $2 --threads $3 --stages $4 \
    --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02t_$cfg.json 2> gpurun_out/r02t_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02t_$cfg.json').readline()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel'])" 2>&1 | tail -1)"
done
