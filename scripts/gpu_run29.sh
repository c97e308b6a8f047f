# new default launch config (PIPE T=128, 2 lanes): parity in that config, default line, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -k "cfg2_full_size or pdec_full_size" > gpurun_out/pytest29.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest29.log
timeout 600 python bench.py > gpurun_out/bench29.json 2> gpurun_out/bench29.err; echo "bench rc=$?"; cat gpurun_out/bench29.json
timeout 600 python bench.py --workload pdec --no-cpu-baseline > gpurun_out/bench29_pdec.json 2>> gpurun_out/bench29.err; echo "pdec rc=$?"; cut -c1-300 gpurun_out/bench29_pdec.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches29.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu29a.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof_pipe_l2 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu29b.log 2>&1; echo "ncu full rc=$?"
