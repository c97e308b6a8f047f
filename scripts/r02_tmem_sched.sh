# round 2: TMEM interpreter batch scheduler knobs (critical-path priority XSLP_TMEM_HEIGHT, window
# XSLP_TMEM_WINDOW, constant-slot recycling XSLP_TMEM_RECYCLE, ops per batch XSLP_TMEM_BATCH):
# GPU parity subset, then bench lines per knob set.  KNOBS="name:VAR=v,VAR=v name2:..." WLS="cfg2 ..."
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_gpu.py -q -x -k "tmem or interp" > gpurun_out/r02ts_pytest.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/r02ts_pytest.log)"
fi
for kn in ${KNOBS:-"old:XSLP_TMEM_RECYCLE=0,XSLP_TMEM_HEIGHT=0,XSLP_TMEM_WINDOW=48" "default:"}; do
  name=${kn%%:*}; envs=$(echo ${kn#*:} | tr ',' ' ')
  for w in ${WLS:-cfg2 pdec cfg3}; do
    env $envs timeout 600 python bench.py --workload $w --kernel interp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/r02ts_${name}_$w.json 2> gpurun_out/r02ts_${name}_$w.err
    echo "$name $w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02ts_${name}_$w.json').readline()); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
