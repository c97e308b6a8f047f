cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cuda_graph or syndrome_full" 2>&1 | tail -2
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["cuda_graph"], d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for w in cfg3 cfg5h; do echo "== $w"; timeout 600 python bench.py --workload $w --no-e2e --no-cpu-baseline 2>/dev/null | tee gpurun_out/bench112_$w.json | python -c "$J"; done
