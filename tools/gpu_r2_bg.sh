cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/exp_plugin_c5.py 4 5 6 8 12 > gpurun_out/r2bg_plugin_c5.log 2>&1
timeout 1500 python tools/exp_plugin_c5.py 4 5 6 8 12 > gpurun_out/r2bg_plugin_c5_b.log 2>&1
