cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "2 0.33" "3 0.35" "3 0.5" "4 0.5" "2 0.5"; do
  set -- $v
  timeout 600 python tools/exp_shards.py 5 8 $1 $2 > gpurun_out/r2_shards_sweep_$1_$2.log 2>&1
done
