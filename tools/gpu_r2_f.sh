cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu_f.log 2>&1; echo pytest=$?
timeout 300 python tools/profile_plugin.py 2 > gpurun_out/r2_profile_plugin_c2.log 2>&1
TB_PIPE_TRACE=1 timeout 300 python tools/profile_plugin.py 2 > gpurun_out/r2_profile_plugin_c2_trace.log 2>&1
timeout 300 python tools/profile_plugin.py 1 > gpurun_out/r2_profile_plugin_c1.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5_v4.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:finalize -c 3 --csv --log-file gpurun_out/r2_fin_c5.csv \
   python tools/run_path.py --config 5 --reps 2 > gpurun_out/r2_ncu_fin.log 2>&1; echo done
