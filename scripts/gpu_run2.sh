# round-1 call 2: parity tests, default bench, variant sweep, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --warmup 3"
for t in 128 256 512; do for l in 1 2 4; do
  echo "== threads $t lanes $l"; $B --threads $t --lanes $l 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['config']['slp']['regs'], d['config']['slp']['spill_bytes'], d['clocks'])"
done; done
for c in none repair; do echo "== compress $c"; $B --compress $c 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['config']['slp'])"; done
for t in 64 128 256; do echo "== interp threads $t"; $B --kernel interp --threads $t 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"; done
for t in 64 128; do echo "== cfg3 threads $t"; $B --workload cfg3 --threads $t 2> gpurun_out/cfg3_$t.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['compile_s'])"; done
echo "== cfg5"; $B --workload cfg5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['config']['slp'])"
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$C > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xslp_sl -s 2 -c 1 -o gpurun_out/prof_sl $C > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
