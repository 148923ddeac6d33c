cd $GRAFT_REPO_ROOT
TB_EXP_FUSED_SERIAL=1 timeout 900 python tools/exp_fused.py > gpurun_out/exp_fused.log 2>&1; echo ex=$?
