cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WJ=33554432,67108864,134217728,268435456 timeout 1200 python tools/exp_plugin_c5.py 1000000 10 1 > gpurun_out/r2ag_plugin_c5.log 2>&1; echo exp=$?
