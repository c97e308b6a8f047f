# round 2: fused multi-program kernels with T+32 <= 256 threads (2 warps per SMSP -> 255 registers)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS}; do
  set -- $(echo $cfg | tr _ " ")
  timeout 900 python bench.py --workload $1 --kernel $2 --threads $3 --lanes $4 --stages $5 --per-module $6 \
    --phases $7 --graph 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02m2_$cfg.json 2> gpurun_out/r02m2_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02m2_$cfg.json').readline()); print(d['value'], d['roofline']['frac'], d['config'].get('multi'))" 2>&1 | tail -1)"
done
