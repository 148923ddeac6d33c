# Expander thread: engine GPU tests, then the config-5 plugin breakdown per record-path mix.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_engine.py -q -x --timeout 900 > gpurun_out/r2af_pt_engine.log 2>&1; echo pt=$?
timeout 900 python tools/exp_plugin_c5.py 1000000 20 10 6 4 > gpurun_out/r2af_plugin_c5.log 2>&1; echo exp=$?
