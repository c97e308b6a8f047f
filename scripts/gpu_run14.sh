# peer (cross-GPU decode) tests on one GPU, xdec benches at N=1, cfg5d stage/thread sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "peer" > gpurun_out/pytest14.log 2>&1
echo "pytest rc=$?"; tail -30 gpurun_out/pytest14.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], d["config"].get("cuda_graph"), {k:d["config"]["slp"][k] for k in ("xor_count","n_instr","maxlive","regs","regs_pipe","spill_bytes","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"], (d.get("e2e") or {}).get("value"), d["roofline"].get("nvlink"))'
for w in xdec1 xdec; do
  echo "== $w"; timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/$w.err | python -c "$J"; tail -3 gpurun_out/$w.err
done
for cfg in "--threads 96 --stages 3" "--threads 64 --stages 4" "--threads 64 --stages 3" "--threads 128 --stages 2 --lanes 1" "--threads 32 --stages 6"; do
  echo "== cfg5d pipe $cfg"; timeout 600 python bench.py --workload cfg5d --kernel pipe $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/cfg5d.err | python -c "$J"
done
for cfg in "--threads 96 --stages 3" "--threads 64 --stages 4" "--threads 128 --stages 2"; do
  echo "== cfg5 pipe $cfg"; timeout 600 python bench.py --workload cfg5 --kernel pipe $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/cfg5.err | python -c "$J"
done
