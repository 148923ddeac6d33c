cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/exp_dispatch.py > gpurun_out/r2at_dispatch.log 2>&1; echo d=$?
