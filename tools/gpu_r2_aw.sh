cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" libtaub200_nopool.so; do
  echo "== variant ${v:-pool} rep $rep" >> gpurun_out/r2aw_plugin_c5.log
  TB_LIB_VARIANT=$v timeout 1200 python tools/exp_plugin_c5.py 6 >> gpurun_out/r2aw_plugin_c5.log 2>&1; echo exp=$?
done
done
