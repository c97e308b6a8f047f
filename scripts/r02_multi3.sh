# round 2: the M^-1 multi-program path as the cfg3 line (and cfg5h --kernel multi): parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "full_size_bench_config" > gpurun_out/r02m3_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02m3_pytest.log
for a in "cfg3" "cfg5h --kernel multi" "cfg3 --kernel syndrome" "cfg5h"; do
  tag=$(echo $a | tr -d ' -')
  timeout 900 python bench.py --workload $a --steps 10 --warmup 3 --no-e2e > gpurun_out/r02m3_$tag.json 2> gpurun_out/r02m3_$tag.err
  echo "$a rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/r02m3_$tag.json').readline()); print(d['value'], d['roofline']['frac'], d['config']['kernel'], d['config']['threads'], d['config'].get('multi'))" 2>&1 | tail -1)"
done
