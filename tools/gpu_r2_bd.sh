cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py -q -x -k "compact or concurrent or sink" > gpurun_out/r2bd_pt.log 2>&1; echo pt=$?
for rep in 1 2; do
for b in 0 1 2 3; do
  echo "== TB_RECORDS_BACKLOG=$b rep $rep" >> gpurun_out/r2bd_plugin_c5.log
  TB_RECORDS_BACKLOG=$b timeout 1200 python tools/exp_plugin_c5.py 6 >> gpurun_out/r2bd_plugin_c5.log 2>&1
done
done
