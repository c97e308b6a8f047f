# BASELINE configs[3]: RS(10,p), p in {2,3,4} x block {64K,256K,1M,4M} x {naive, RePair, XorRePair+fuse+DFS}
# (10 GiB of data per point).  Output: one JSON line per point in gpurun_out/cfg4.jsonl
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/cfg4.jsonl
for p in 2 3 4; do for b in 65536 262144 1048576 4194304; do for c in none repair xorrepair; do
  extra=""
  if [ $c = repair ]; then extra="--fuse 0 --schedule 0"; fi   # RePair alone: binary, creation order
  timeout 300 python bench.py --workload cfg4 --p $p --block-bytes $b --compress $c $extra --no-e2e --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null >> gpurun_out/cfg4.jsonl || echo "{\"failed\": \"p=$p b=$b c=$c\"}" >> gpurun_out/cfg4.jsonl
done; done; done
python scripts/cfg4_table.py gpurun_out/cfg4.jsonl
