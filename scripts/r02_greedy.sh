# round 2: NEXT #2 on the device -- greedy-schedule parity tests, then DFS vs greedy GB/s on
# RS(20,4) decode (cfg5d) through the LDG straight-line kernel and the PIPE kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py -q -x -k "greedy or random_programs" > gpurun_out/r02g_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02g_pytest.log
for k in "straight 128" "pipe 256"; do
  set -- $k
  for sc in "1 64" "2 16" "2 64" "2 512"; do
    set -- $k $sc
    timeout 600 python bench.py --workload cfg5d --kernel $1 --threads $2 --schedule $3 --greedy-capacity $4 \
      --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02g_$1_$3_$4.json 2> gpurun_out/r02g_$1_$3_$4.err
    echo "$1 T=$2 sched=$3 cap=$4 rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02g_$1_$3_$4.json').readline()); print(d['value'], d['roofline']['frac'], d['config']['slp']['regs'], d['config']['slp']['spill_bytes'], d['config']['slp']['regs_pipe'], d['config']['slp']['spill_bytes_pipe'])" 2>&1 | tail -1)"
  done
done
