# round-1 call 3: tests incl. TMA + grouped decode; sweep TMA variants; ncu on the TMA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --warmup 3"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], {k:d["config"]["slp"][k] for k in ("regs","spill_bytes","regs_tma","spill_bytes_tma")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("compile_s"))'
for w in cfg2 cfg5; do for k in straight tma; do for t in 64 128 256; do
  echo "== $w $k threads $t"; $B --workload $w --kernel $k --threads $t 2>gpurun_out/err_${w}_${k}_$t.log | python -c "$J"
done; done; done
echo "== cfg2 tma lanes2 t128"; $B --kernel tma --lanes 2 --threads 128 2>/dev/null | python -c "$J"
echo "== cfg2 tma lanes2 t64"; $B --kernel tma --lanes 2 --threads 64 2>/dev/null | python -c "$J"
echo "== cfg2 none tma t128"; $B --kernel tma --compress none --threads 128 2>/dev/null | python -c "$J"
echo "== cfg2 none straight t128"; $B --kernel straight --compress none --threads 128 2>/dev/null | python -c "$J"
for k in grouped grouped_tma interp; do for t in 64 128; do
  echo "== cfg3 $k threads $t"; $B --workload cfg3 --kernel $k --threads $t 2>gpurun_out/err_cfg3_${k}_$t.log | python -c "$J"
done; done
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --kernel tma --threads 128"
$C > gpurun_out/ncu_plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $C > gpurun_out/ncu_launch3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xslp_sl -s 2 -c 1 -o gpurun_out/prof_tma $C > gpurun_out/ncu_full3.log 2>&1
echo "ncu rc=$?"
