# approach (1) kernel with 3-group 8-entry PRMT tables: parity, bench cfg2t, ncu ALU-pipe counts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "gf_table" 2>&1 | tail -2
J='import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
timeout 600 python bench.py --workload cfg2t --no-e2e --no-cpu-baseline 2>gpurun_out/s83.err | tee gpurun_out/bench83_cfg2t.json | python -c "$J"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed.sum,smsp__inst_executed_op_shared_ld.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gftable -s 3 -c 1 --csv python bench.py --workload cfg2t --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu83_cfg2t.csv 2>gpurun_out/ncu83.err; echo "ncu rc=$?"
grep -v "^==" gpurun_out/ncu83_cfg2t.csv | tail -12
