cd $GRAFT_REPO_ROOT
for sl in 0 1; do
  TB_PLAN_SLICE=$sl TB_TRACE=1 timeout 300 python tools/exp_epi.py 2 3 > gpurun_out/exp_slice_$sl.log 2>&1
  echo "slice=$sl $(grep 'gemm ms' gpurun_out/exp_slice_$sl.log | tr '\n' ' ')"
done
TB_PLAN_SLICE=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest_slice.log 2>&1; echo pytest=$?
