# round 2: ncu --set full of one pipelined-interpreter launch (cfg2 by default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${W:-cfg2}; T=${T:-256}; L=${L:-1}; S=${S:-2}; TAG=${TAG:-r02_interp_cfg2}
ncu --set full --clock-control none --import-source on -k regex:xslp_interp_pipe -s 2 -c 1 \
  -o gpurun_out/$TAG -f python bench.py --workload $W --kernel interp --threads $T --lanes $L --stages $S \
  --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}.log
