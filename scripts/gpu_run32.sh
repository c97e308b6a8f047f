# full GPU suite with auto input phases; cfg5 / cfg5d default lines; ncu of the phased kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke32.log 2>&1; echo "smoke rc=$?"
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest32.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest32.log
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 3 > gpurun_out/bench32_cfg5.json 2> gpurun_out/bench32.err; echo "cfg5 rc=$?"; cut -c1-200 gpurun_out/bench32_cfg5.json
timeout 900 python bench.py --workload cfg5d --steps 20 --warmup 3 > gpurun_out/bench32_cfg5d.json 2>> gpurun_out/bench32.err; echo "cfg5d rc=$?"; cut -c1-200 gpurun_out/bench32_cfg5d.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_pipe -s 3 -c 1 -o gpurun_out/prof_cfg5_phases python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu32.log 2>&1; echo "ncu rc=$?"
