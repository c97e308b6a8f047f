# round-1 call 4: interpreter v2 parity + speed; P_dec single-pattern; ncu on cfg5 / pdec kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
B="timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --warmup 3"
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], {k:d["config"]["slp"][k] for k in ("regs","spill_bytes","regs_tma","spill_bytes_tma")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("compile_s"))'
for t in 64 128 256; do echo "== cfg2 interp t$t"; $B --kernel interp --threads $t 2>/dev/null | python -c "$J"; done
for t in 64 128; do echo "== cfg3 interp t$t"; $B --workload cfg3 --kernel interp --threads $t 2>gpurun_out/err4_cfg3_$t.log | python -c "$J"; done
for k in straight tma interp; do for t in 64 128; do echo "== pdec $k t$t"; $B --workload pdec --kernel $k --threads $t 2>/dev/null | python -c "$J"; done; done
echo "== cfg3 grouped t64 streams 16"; $B --workload cfg3 --kernel grouped --threads 64 --streams 16 2>/dev/null | python -c "$J"
echo "== cfg3 grouped t64 streams 4"; $B --workload cfg3 --kernel grouped --threads 64 --streams 4 2>/dev/null | python -c "$J"
C5="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workload cfg5 --threads 64"
CP="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workload pdec --threads 128"
$C5 --kernel tma > gpurun_out/ncu4_plain1.log 2>&1 && $C5 --kernel straight > gpurun_out/ncu4_plain2.log 2>&1 && \
$CP --kernel tma > gpurun_out/ncu4_plain3.log 2>&1 && $CP --kernel interp > gpurun_out/ncu4_plain4.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp -s 2 -c 1 -o gpurun_out/prof4_cfg5_tma $C5 --kernel tma > gpurun_out/ncu4_a.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp -s 2 -c 1 -o gpurun_out/prof4_cfg5_ldg $C5 --kernel straight > gpurun_out/ncu4_b.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp -s 2 -c 1 -o gpurun_out/prof4_pdec_tma $CP --kernel tma > gpurun_out/ncu4_c.log 2>&1 && \
ncu --set full --clock-control none -k regex:xslp -s 2 -c 1 -o gpurun_out/prof4_pdec_interp $CP --kernel interp > gpurun_out/ncu4_d.log 2>&1
echo "ncu rc=$?"
