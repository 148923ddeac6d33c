# (Reverted experiment: the packed plan and TB_NO_PACKED_PLAN are in git history.) GEMM plan comparison on configs 2 and 3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 3; do
python tools/exp_splits_c2.py $c > gpurun_out/gemm_c$c.log 2>&1
TB_NO_PACKED_PLAN=1 python tools/exp_splits_c2.py $c > gpurun_out/gemm_c${c}_rr.log 2>&1
done
TB_TRACE=1u python tools/exp_splits_c2.py 2 > gpurun_out/gemm_c2_trace.log 2>&1
