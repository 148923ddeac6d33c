cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 900 -k "finalize or full_counts or config5" > gpurun_out/r2_pytest_gpu_h.log 2>&1; echo pytest=$?
timeout 900 python tools/exp_shards.py 5 8 > gpurun_out/r2_shards_c5.log 2>&1; echo shards=$?
timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:finalize -c 1 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_fin_c5_v2.csv 2>&1; echo ncu=$?
