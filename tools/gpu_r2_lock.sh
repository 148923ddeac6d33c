# K-lockstep throttle sweep on config 5 (time + clocks + power), then DRAM bytes per band
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "16 4 0 0" "16 4 16 0" "16 4 64 4" "16 4 64 10" "16 4 128 10" "16 4 32 18" "16 4 0 0"; do
  set -- $v
  TB_GEMM_GR=$1 TB_GEMM_WIN=$2 TB_GEMM_LEAD=$3 TB_GEMM_LAGQ=$4 timeout 300 python tools/exp_unit_order.py 6 >> gpurun_out/r2_lock2.log 2>&1
done
