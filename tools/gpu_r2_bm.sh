cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for fw in 134217728 33554432 8388608; do
  echo "== TB_FIRST_WINDOW_JOBS=$fw rep $rep" >> gpurun_out/r2bm_plugin_c5.log
  TB_FIRST_WINDOW_JOBS=$fw timeout 1200 python tools/exp_plugin_c5.py 6 >> gpurun_out/r2bm_plugin_c5.log 2>&1
done
done
