# round 2: ncu of one TMEM-interpreter launch (cfg2 by default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WL=${WL:-cfg2}
ARGS="--workload $WL --kernel interp --interp tmem --lanes 2 --threads 128 --stages 2 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/r02tn_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xslp_interp_tmem -s 2 -c 1 \
  -o gpurun_out/r02_tmem_$WL -f python bench.py $ARGS > gpurun_out/r02_tmem_ncu.log 2>&1
echo "ncu rc=$?"
