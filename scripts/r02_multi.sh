# round 2: the configured heterogeneous decode (M^-1 program per erasure pattern, fused multi-program
# kernels) on cfg3 / cfg5h: launch sweep, then ncu of one cfg5h module launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS:-cfg3_256_1_2_20_0 cfg3_128_2_2_20_0 cfg3_256_1_3_20_0 cfg5h_256_1_2_20_2 cfg5h_256_1_3_10_6 cfg5h_256_1_2_10_2}; do
  set -- $(echo $cfg | tr _ " ")
  timeout 900 python bench.py --workload $1 --kernel multi --threads $2 --lanes $3 --stages $4 --per-module $5 \
    --phases $6 --graph 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02m_$cfg.json 2> gpurun_out/r02m_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02m_$cfg.json').readline()); print(d['value'], d['roofline']['frac'], d['config'].get('multi'))" 2>&1 | tail -1)"
done
if [ -n "$NCU" ]; then
  set -- $(echo $NCU | tr _ " ")
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 5 -c 1 \
    -o gpurun_out/r02m_ncu_$NCU -f python bench.py --workload $1 --kernel multi --threads $2 --lanes $3 --stages $4 \
    --per-module $5 --phases $6 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02m_ncu.log 2>&1
  echo "ncu rc=$?"
fi
