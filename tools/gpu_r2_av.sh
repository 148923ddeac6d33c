cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/probe_expand.py > gpurun_out/r2av_probe_expand.log 2>&1; echo probe=$?
timeout 1200 python tools/exp_plugin_c5.py 6 5 4 > gpurun_out/r2av_plugin_c5.log 2>&1; echo exp=$?
