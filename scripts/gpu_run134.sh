# (re-run of gpu_run101 with the final code) control-flow check of bench.py's N>1 path on the one-GPU box: torchrun with 2 ranks sharing
# cuda:0 (XSLP_BENCH_SHARED_GPU=1: gloo barriers / max over ranks; ranks never wait on each
# other's kernels).  Exit codes and the JSON line's shape are the result, not the numbers.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=29611
for w in cfg2 cfg3 cfg5 xdec xdec1; do
  P=$((P+1))
  XSLP_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload $w --steps 3 --warmup 3 \
    > gpurun_out/mr134_$w.json 2> gpurun_out/mr134_$w.err
  echo "$w rc=$? lines=$(grep -c '^{' gpurun_out/mr134_$w.json)"
  python -c "import json; d=json.loads(open('gpurun_out/mr134_$w.json').readline()); print(d['n_gpus'], d['scaling'], d['config']['parallelism'], d['value'], d['gpu_launches'], (d.get('e2e') or {}).get('value'), d.get('cpu_baseline'))" 2>&1 | tail -1
done
