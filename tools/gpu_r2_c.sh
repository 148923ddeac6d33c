cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_d2h_sustained.py > gpurun_out/r2_d2h_sustained.log 2>&1; echo d2h=$?
timeout 1200 python tools/exp_dispatch.py > gpurun_out/r2_dispatch.log 2>&1; echo dispatch=$?
bash tools/gpu_r2_unitorder.sh; echo unitorder=$?
