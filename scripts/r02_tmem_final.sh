# round 2: the TMEM interpreter at its defaults (--kernel interp): bench lines + ncu of cfg2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg2 pdec cfg3 cfg5; do
  timeout 600 python bench.py --workload $w --kernel interp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02tf_$w.json 2> gpurun_out/r02tf_$w.err
  echo "$w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02tf_$w.json').readline()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel'], d['config'].get('threads'), d['config'].get('stages'))" 2>&1 | tail -1)"
done
[ -n "$NONCU" ] || { ARGS="--workload cfg2 --kernel interp --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:xslp_interp_tmem -s 2 -c 1 \
  -o gpurun_out/r02_tmem_final_cfg2 -f python bench.py $ARGS > gpurun_out/r02tf_ncu.log 2>&1; echo "ncu rc=$?"; }
