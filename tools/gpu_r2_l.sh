cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "3 0.5" "2 0.5" "3 0.35"; do
  set -- $v
  timeout 600 python tools/exp_shards.py 5 8 $1 $2 > gpurun_out/r2_shards_aligned_$1_$2.log 2>&1
done
