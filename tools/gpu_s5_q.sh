# session 5: row bands per config-5 step with the lockstep throttle (8 was tuned without it)
mkdir -p gpurun_out
L=gpurun_out/s5q_bands.log; : > $L
for gb in 8 1 2 4 16 8; do GB=$gb timeout 300 python tools/exp_unit_order.py 6 >> $L 2>&1; done
cat $L
