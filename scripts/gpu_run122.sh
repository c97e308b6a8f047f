# ncu --set full of the current syndrome-form kernels (cfg3: reuse 40, 16 per module; cfg5h: reuse 16, 10 per module)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg3 cfg5h; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_multi -s 60 -c 1 -o gpurun_out/prof122_$w python bench.py --workload $w --graph 0 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/s122_$w.err; echo "$w rc=$?"
done
