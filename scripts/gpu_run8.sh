# round-1 call 8: byte layout + codec parity; byte-layout bench; default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu8.log
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["kernel"], {k:d["config"]["slp"][k] for k in ("regs","regs_pipe")}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for t in 64 128 256; do echo "== cfg2b t$t"; timeout 300 python bench.py --workload cfg2b --threads $t --no-e2e --no-cpu-baseline --steps 30 --warmup 3 2>/dev/null | python -c "$J"; done
echo "== default"; timeout 900 python bench.py > gpurun_out/bench8_default.json 2>gpurun_out/bench8_default.err; python -c "$J" < gpurun_out/bench8_default.json
