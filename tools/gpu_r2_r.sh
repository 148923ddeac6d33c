cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 100 30 60 200; do
  TB_PLAN_EPI=$e timeout 300 python tools/exp_splits.py 2 >> gpurun_out/r2_splits_c2.log 2>&1
done
TB_PLAN_EPI=100 timeout 300 python tools/exp_splits.py 3 >> gpurun_out/r2_splits_c3.log 2>&1
