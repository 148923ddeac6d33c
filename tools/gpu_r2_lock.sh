# K-lockstep throttle sweep on config 5 (time + clocks + power), then DRAM bytes per band
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "8 8 0" "8 8 64" "16 4 0" "16 4 32" "16 4 64" "16 4 128" "16 4 256" "8 8 128" "16 4 0"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_LEAD=$3 timeout 300 python tools/exp_unit_order.py 6 >> gpurun_out/r2_lock.log 2>&1
done
for v in "16 4 0" "16 4 64" "16 4 256"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_LEAD=$3 timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_LEAD=$3 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
     -k regex:gemm_fp4 -c 8 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_lock_ncu_$1_$2_$3.csv 2>&1
done
