cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "12 4" "12 8" "8 8" "14 8"; do
  set -- $cfg
  echo "== TB_EXPAND_THREADS=$1 TB_PASS_SLOTS=$2" >> gpurun_out/r2ae_plugin_c5_b.log
  TB_EXPAND_THREADS=$1 TB_PASS_SLOTS=$2 timeout 900 python tools/exp_plugin_c5.py 1000000 10 >> gpurun_out/r2ae_plugin_c5_b.log 2>&1; echo exp=$?
done
