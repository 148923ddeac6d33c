# Round 2, first call: the config-5 headline bench line, its launch list, and one ncu --set full capture of
# a config-5 GEMM row-band launch (roofline.traffic).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo bench=$?
timeout 600 python tools/run_path.py --config 5 --reps 2 > gpurun_out/r2_plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv \
    python tools/run_path.py --config 5 --reps 2 > gpurun_out/r2_ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -c 1 \
    -o gpurun_out/r2_c5_gemm python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_ncu_full.log 2>&1; echo ncufull=$?
