# session 5: K-lockstep throttle with the warp-parallel poll, both operand codings (config 5: time, clock, power)
mkdir -p gpurun_out
L=gpurun_out/s5f_lockstep.log; : > $L
for v in "1 0" "1 32" "1 64" "1 128" "1 256" "1 16" "0 64" "0 0" "1 0"; do
  set -- $v
  echo "TB_SIGN_OFS=$1" >> $L
  TB_SIGN_OFS=$1 TB_GEMM_LEAD=$2 timeout 300 python tools/exp_unit_order.py 6 >> $L 2>&1
done
cat $L
