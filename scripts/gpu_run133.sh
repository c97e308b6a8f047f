# long sustained default line (20000 steps, ~45 s) under the power cap
cd $GRAFT_REPO_ROOT
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["clocks"]; s=d["step_ms"]; print(d["steps"], d["value"], d["roofline"]["frac"], s, c["sm_mhz"], c["power_w"], c["reasons"], c["samples"])'
timeout 900 python bench.py --steps 20000 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tee gpurun_out/bench133_long.json | python -c "$J"
