cd $GRAFT_REPO_ROOT
timeout 900 python tools/exp_fp8.py > gpurun_out/exp_fp8.log 2>&1; echo exp=$?
