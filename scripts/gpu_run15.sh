# PIPE consumer groups: parity tests, then sweeps on RS(20,4) (cfg5, cfg5d) and RS(10,4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "consumer_groups or cfg5_full_chunk or test_cfg2_full_size" > gpurun_out/pytest15.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest15.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["threads"], c["stages"], c["groups"], {k:c["slp"][k] for k in ("xor_count","group_xor","regs_pipe","spill_bytes_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg5 cfg5d; do
for cfg in "--threads 128 --groups 1" "--threads 128 --groups 2" "--threads 96 --groups 2" "--threads 64 --groups 3" "--threads 64 --groups 4" "--threads 96 --groups 3"; do
  echo "== $w $cfg"; timeout 600 python bench.py --workload $w --kernel pipe --stages 2 $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep15.err | python -c "$J"
done; done
for w in cfg2 pdec; do
for cfg in "--threads 256 --groups 1" "--threads 128 --groups 2" "--threads 256 --groups 2" "--threads 128 --groups 3"; do
  echo "== $w $cfg"; timeout 600 python bench.py --workload $w --kernel pipe --stages 2 $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep15.err | python -c "$J"
done; done
