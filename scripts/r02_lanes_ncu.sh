# round 2: ncu of one lane-interpreter launch (cfg2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out

T=${T:-512}
timeout 300 python bench.py --workload cfg2 --kernel interp --threads $T --stages 2 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02ln_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xslp_interp_lanes -s 2 -c 1 \
  -o gpurun_out/r02_lanes_cfg2 -f python bench.py --workload cfg2 --kernel interp --threads $T --stages 2 \
  --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02_lanes_ncu.log 2>&1
echo "ncu rc=$?"
