cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_engine.py -q -x --timeout 900 > gpurun_out/r2bf_pt.log 2>&1; echo pt=$?
for rep in 1 2; do
for c in 1 0; do
  echo "== TB_COMPACT_NUM=$c rep $rep" >> gpurun_out/r2bf_plugin_c5.log
  TB_COMPACT_NUM=$c timeout 1200 python tools/exp_plugin_c5.py 6 1000000 >> gpurun_out/r2bf_plugin_c5.log 2>&1
done
done
