# GEMM unit-order sweep on config 5 (time + clocks), then DRAM bytes of band 0 for each variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "8 8 0" "8 8 1" "16 4 0" "16 4 1" "4 16 0" "32 2 1" "16 8 1" "8 4 1"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_SERP=$3 timeout 300 python tools/exp_unit_order.py 6 >> gpurun_out/r2_unitorder.log 2>&1
done
for v in "8 8 0" "16 4 1" "32 2 1"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_SERP=$3 timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_SERP=$3 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
     -k regex:gemm_fp4 -c 8 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_unitorder_ncu_$1_$2_$3.csv 2>&1
done
