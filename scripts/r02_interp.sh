# round 2: pipelined interpreter (paired micro-ops, software-pipelined operand loads) -- parity + sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests/test_gpu.py -x -q -k "interp or heterogeneous or random" > gpurun_out/r02i_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02i_pytest.log
for cfg in ${CFGS:-cfg2_256_1_2 pdec_256_1_2 cfg3_256_1_2}; do
  set -- $(echo $cfg | tr _ " ")
  timeout 300 python bench.py --workload $1 --kernel interp --threads $2 --lanes $3 --stages $4 --steps 5 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/r02i_$1_$2_$3_$4.json 2> gpurun_out/r02i_$1_$2_$3_$4.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02i_$1_$2_$3_$4.json').readline()); print(d['value'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
