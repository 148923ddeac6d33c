cd $GRAFT_REPO_ROOT
timeout 900 python tools/exp_bands.py 3 > gpurun_out/exp_bands.log 2>&1; echo ex=$?
