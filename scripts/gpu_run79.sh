# cfg5h / cfg3 syndrome-form: 2 words per thread (halves instruction bytes per data byte)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
J='import json,sys; d=json.loads(sys.stdin.read()); c=d["config"]; print(d["value"], d["roofline"]["frac"], c["multi"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])'
for a in "--distinct 1" ""; do
for k in "--threads 128 --phases 6 --lanes 2" "--threads 128 --phases 4 --lanes 2" "--threads 128 --phases 3 --lanes 2" "--threads 64 --phases 6 --lanes 2 --stages 3" "--threads 256 --phases 6 --lanes 2" "--threads 256 --phases 6" "--threads 128"; do
  echo "== cfg5h $a $k"
  timeout 600 python bench.py --workload cfg5h --kernel syndrome --per-module 16 $a $k --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s79.err | python -c "$J"
done; done
for k in "--threads 128 --lanes 2" "--threads 128 --lanes 2 --phases 2" "--threads 256 --lanes 2" "--threads 256"; do
  echo "== cfg3 $k"
  timeout 600 python bench.py --workload cfg3 --kernel syndrome --per-module 32 $k --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/s79.err | python -c "$J"
done
