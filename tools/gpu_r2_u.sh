cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2_splits_c2_v4.log 2>&1
TB_GEMM_NO_FIXUP=1 timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2_splits_c2_v4_nofix.log 2>&1
timeout 300 python tools/exp_splits.py 1 > gpurun_out/r2_splits_c1_v4.log 2>&1
TB_GEMM_NO_FIXUP=1 timeout 300 python tools/exp_splits.py 1 > gpurun_out/r2_splits_c1_v4_nofix.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 900 -k "splits or config1 or config2 or small_shapes" > gpurun_out/r2_pytest_gpu_u.log 2>&1; echo pytest=$?
