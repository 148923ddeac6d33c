cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -k "engine or pipeline or full_counts or streams" > gpurun_out/r2_pytest_gpu_d.log 2>&1; echo pytest=$?
timeout 900 python tools/exp_plugin.py 5 > gpurun_out/r2_plugin_c5_v2.log 2>&1; echo plugin=$?
for c in 2 3; do
  for o in "16 4" "8 8"; do
    set -- $o
    TB_GEMM_GR=$1 TB_GEMM_WIN=$2 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --e2e-steps 0 --e2e-tau-steps 2 --no-cpu-baseline > gpurun_out/r2_bench_c${c}_order_$1_$2.json 2>&1
  done
done
bash tools/gpu_r2_lock.sh
