cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu_j.log 2>&1; echo pytest=$?
timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:finalize -c 1 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_fin_c5_v4.csv 2>&1; echo ncu=$?
timeout 900 python tools/exp_shards.py 5 8 > gpurun_out/r2_shards_c5_v3.log 2>&1; echo shards=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5_v5.json 2>&1; echo bench=$?
