# session 5: lockstep lead x unit order (config 5, offset operands)
mkdir -p gpurun_out
L=gpurun_out/s5g_lockstep_order.log; : > $L
for v in "16 4 32" "8 8 32" "32 2 32" "4 16 32" "16 8 32" "16 4 24" "16 4 48" "16 4 32"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_LEAD=$3 timeout 300 python tools/exp_unit_order.py 6 >> $L 2>&1
done
cat $L
