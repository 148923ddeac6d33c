cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -v > gpurun_out/r2_pytest_gpu_e.log 2>&1; echo pytest=$?
timeout 900 python tools/exp_plugin.py 5 > gpurun_out/r2_plugin_c5_v3.log 2>&1; echo plugin=$?
TB_EVENT_POLL=1 timeout 900 python tools/exp_plugin.py 5 > gpurun_out/r2_plugin_c5_v3_poll.log 2>&1; echo plugin=$?
for c in 2 3 1; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --e2e-steps 2 --e2e-tau-steps 5 > gpurun_out/r2_bench_c${c}.json 2>&1
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 > gpurun_out/r2_bench_c4.json 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5_v3.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_v3.csv \
   python bench.py --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/r2_ncu_launch_v3.log 2>&1; echo done
