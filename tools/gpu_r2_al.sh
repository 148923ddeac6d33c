cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 1; do
 for slots in 4 8; do
  echo "== config $c TB_PASS_SLOTS=$slots" >> gpurun_out/r2al_small.log
  CFG=$c TB_PASS_SLOTS=$slots timeout 600 python tools/exp_plugin_c5.py 1 6 1000000 >> gpurun_out/r2al_small.log 2>&1
 done
done
