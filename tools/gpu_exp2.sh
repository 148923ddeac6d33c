cd $GRAFT_REPO_ROOT
for c in 4 8 16 32 64; do TB_EXP_FIN_CPS=$c timeout 300 python tools/exp_fin.py > gpurun_out/exp_fin_$c.log 2>&1; echo "cps=$c $(cat gpurun_out/exp_fin_$c.log | tr '\n' ' ')"; done
