# ALU / LDS microbenchmark (SURVEY 8(d) integer roof) + default bench line with the new roofline keys
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_probe scripts/alu_probe.cu && timeout 120 /tmp/alu_probe | tee gpurun_out/alu_probe81.jsonl
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench81.json 2>gpurun_out/s81.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench81.json')); print(d['value'], d['roofline'])"
