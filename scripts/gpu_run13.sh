# cfg5d (RS(20,4) decode) bench + sweep, cfg3 with/without CUDA graph, new parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cfg5_full_chunk or graph" > gpurun_out/pytest13.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest13.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], d["config"].get("cuda_graph"), {k:d["config"]["slp"][k] for k in ("xor_count","n_instr","maxlive","regs","regs_pipe","spill_bytes","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"], (d.get("e2e") or {}).get("value"))'
for g in 0 1; do for st in 8 16; do
  echo "== cfg3 graph=$g streams=$st"; timeout 600 python bench.py --workload cfg3 --graph $g --streams $st --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/cfg3_$g_$st.err | python -c "$J"
done; done
for cfg in "--kernel pipe --threads 128" "--kernel pipe --threads 64" "--kernel pipe --threads 256" "--kernel straight --threads 64" "--kernel straight --threads 128" "--kernel tma --threads 64"; do
  echo "== cfg5d $cfg"; timeout 600 python bench.py --workload cfg5d $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/cfg5d.err | python -c "$J"
done
echo "== cfg5d default full line"
timeout 900 python bench.py --workload cfg5d --steps 10 --warmup 3 > gpurun_out/bench_cfg5d.json 2>gpurun_out/bench_cfg5d.err; echo rc=$?
cat gpurun_out/bench_cfg5d.json
echo "== pdec default full line"
timeout 900 python bench.py --workload pdec > gpurun_out/bench_pdec.json 2>gpurun_out/bench_pdec.err; echo rc=$?
cat gpurun_out/bench_pdec.json
