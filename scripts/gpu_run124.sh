# codec front end throughput (encode / reconstruct / decode of device data)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/codec_probe.py 2>gpurun_out/s124.err | tee gpurun_out/codec124.jsonl; tail -3 gpurun_out/s124.err
