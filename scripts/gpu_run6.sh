# round-1 call 6: default bench as the driver runs it, torchrun N=1, reference arm, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu6.log
timeout 900 python bench.py > gpurun_out/bench6_default.json 2> gpurun_out/bench6_default.err
echo "bench rc=$?"; cat gpurun_out/bench6_default.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_torchrun.json 2> gpurun_out/bench6_torchrun.err
echo "torchrun rc=$?"; cat gpurun_out/bench6_torchrun.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench6_ref.json 2> gpurun_out/bench6_ref.err
echo "ref rc=$?"; cat gpurun_out/bench6_ref.json
for w in pdec cfg3 cfg5; do timeout 600 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/bench6_$w.json 2>/dev/null; echo "$w rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench6_$w.json')); print(d['value'], d['roofline']['frac'], d['clocks'])"; done
C="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/ncu6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches6.csv $C > gpurun_out/ncu6_launch.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp_sl -s 4 -c 1 -o gpurun_out/prof6_cfg2_pipe $C > gpurun_out/ncu6_full.log 2>&1
echo "ncu rc=$?"
