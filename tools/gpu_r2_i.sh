cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 900 -k "finalize or config1 or config2 or small_shapes or host_entry or streams" > gpurun_out/r2_pytest_gpu_i.log 2>&1; echo pytest=$?
timeout 300 python tools/probe_write_bw.py > gpurun_out/r2_write_bw.log 2>&1; echo bw=$?
timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:finalize -c 1 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_fin_c5_v3.csv 2>&1; echo ncu=$?
timeout 900 python tools/exp_shards.py 5 8 > gpurun_out/r2_shards_c5_v2.log 2>&1; echo shards=$?
