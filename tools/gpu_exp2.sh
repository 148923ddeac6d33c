cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp_splits_c2.py 2 > gpurun_out/exp_splits.log 2>&1; echo ex=$?
