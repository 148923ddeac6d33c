cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
for te in 20 40 70 100; do
  TB_PLAN_TEPI=$te TB_TRACE=1 timeout 300 python tools/exp_epi.py 2 > gpurun_out/exp_te_$te.log 2>&1
  echo "te=$te $(grep plan4 gpurun_out/exp_te_$te.log | head -1) $(grep 'gemm ms' gpurun_out/exp_te_$te.log)"
done
