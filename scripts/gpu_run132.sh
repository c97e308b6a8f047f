# codec: threads of its single-stripe programs (small objects under-fill the GPU at T=128)
cd $GRAFT_REPO_ROOT
for t in 32 64 128 256; do timeout 600 python scripts/codec_probe.py $t 2>&1 | tail -3; done
