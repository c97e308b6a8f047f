# BASELINE configs[0] latency probe (RS(4,2) Cauchy, one 4 x 4 KiB stripe)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/latency_probe.py 2>gpurun_out/s103.err | tee gpurun_out/latency103.jsonl
tail -3 gpurun_out/s103.err
