# M^-1 fused kernels with auto reuse 64: parity (multi tests, heterogeneous fuzz), xdec and cfg3 --kernel multi lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "multi or heterogeneous or peer" 2>&1 | tail -1
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; m=c.get("multi") or {}; print(d["value"], d["roofline"]["frac"], m.get("regs"), c.get("const_reuse"), d["clocks"]["sm_mhz"])'
for w in "xdec" "cfg3 --kernel multi --threads 256"; do
  echo "== $w"; timeout 600 python bench.py --workload $w --no-e2e --no-cpu-baseline 2>>gpurun_out/s110.err | tee gpurun_out/bench110.json | python -c "$J"
done
