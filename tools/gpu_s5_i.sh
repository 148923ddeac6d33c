# session 5: ncu --set full of the GEMM with lockstep + offset operands (config 5 band 0, config 3), launch list of the bench command
mkdir -p gpurun_out
python tools/run_path.py --config 5 --reps 1 > gpurun_out/s5i_plain5.log 2>&1; echo plain5=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -c 1 -o gpurun_out/s5i_c5_gemm -f \
    python tools/run_path.py --config 5 --reps 1 > gpurun_out/s5i_ncu5.log 2>&1; echo ncu5=$?
timeout 900 ncu --set full --clock-control none -k regex:gemm_fp4 -s 2 -c 1 -o gpurun_out/s5i_c3_gemm -f \
    python tools/run_path.py --config 3 --reps 3 > gpurun_out/s5i_ncu3.log 2>&1; echo ncu3=$?
python bench.py --steps 2 --warmup 3 > gpurun_out/s5i_b.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5i_launches_config5.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/s5i_ncu_launches.log 2>&1; echo launches=$?
ncu -i gpurun_out/s5i_c5_gemm.ncu-rep --page raw --csv > gpurun_out/s5i_c5_gemm_raw.csv 2>/dev/null
ncu -i gpurun_out/s5i_c3_gemm.ncu-rep --page raw --csv > gpurun_out/s5i_c3_gemm_raw.csv 2>/dev/null
ls -la gpurun_out/s5i_*
