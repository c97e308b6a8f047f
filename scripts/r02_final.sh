# round 2 regression: smoke, the full -m gpu suite, every workload's bench line (20 steps),
# the reference arm, the 2-rank control-flow check (one GPU, shared), the ncu launch list of the
# default command and one `ncu --set full` of the default kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"
if [ -z "$NOTEST" ]; then
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r02f_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02f_pytest.log
fi
for w in ${WLS:-cfg2 pdec cfg3 cfg5 cfg5d cfg5h cfg2b cfg2t xdec1 xdec}; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/r02f_$w.json 2> gpurun_out/r02f_$w.err
  echo "$w rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02f_$w.json').readline()); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'], (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02f_reference.json 2> gpurun_out/r02f_reference.err
echo "reference rc=$? $(head -c 300 gpurun_out/r02f_reference.json)"
XSLP_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --workload cfg2 --steps 3 --warmup 3 --no-e2e \
  > gpurun_out/r02f_2rank_cfg2.json 2> gpurun_out/r02f_2rank_cfg2.err
echo "2-rank (shared GPU) rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02f_2rank_cfg2.json').readline()); print(d['n_gpus'], d['config']['parallelism'], [r['gbs'] for r in d['per_rank']])" 2>&1 | tail -1)"
if [ -z "$NONCU" ]; then
  timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_launch.log 2>&1
  echo "ncu launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 \
    -o gpurun_out/r02f_default_full -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02f_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
