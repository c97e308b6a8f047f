# round-1 call 5: persistent TMA pipeline kernel: bounded smoke, parity, sweep, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python scripts/pipe_smoke.py > gpurun_out/pipe_smoke.log 2>&1; rc=$?
echo "pipe smoke rc=$rc"; cat gpurun_out/pipe_smoke.log | tail -3
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu5.log
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --warmup 3"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], {k:d["config"]["slp"][k] for k in ("regs","regs_tma","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg2 pdec cfg5; do for t in 64 128 256; do for st in 2 3 4; do
  echo "== $w pipe threads $t stages $st"; $B --workload $w --kernel pipe --threads $t --stages $st 2>/dev/null | python -c "$J"
done; done; done
for t in 64 128; do echo "== cfg3 grouped_pipe t$t"; $B --workload cfg3 --kernel grouped_pipe --threads $t --streams 4 2>/dev/null | python -c "$J"; done
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workload cfg5 --kernel pipe --threads 128 --stages 2"
$C > gpurun_out/ncu5_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp_sl -s 2 -c 1 -o gpurun_out/prof5_cfg5_pipe $C > gpurun_out/ncu5.log 2>&1
echo "ncu rc=$?"
