# GF-table (approach (1)) kernel: parity + bench vs the XOR-SLP byte layout (cfg2b); ncu of both
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "gf_table" > gpurun_out/pytest21.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest21.log
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], c["threads"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"])'
for w in cfg2t cfg2b; do
  echo "== $w"; timeout 900 python bench.py --workload $w --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/sweep21.err | python -c "$J"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gftable -s 3 -c 1 -o gpurun_out/prof_gftable python bench.py --workload cfg2t --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu21a.log 2>&1; echo "a rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xslp_sl_batch -s 3 -c 1 -o gpurun_out/prof_byte python bench.py --workload cfg2b --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu21b.log 2>&1; echo "b rc=$?"
