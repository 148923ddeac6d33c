# session 5: final-state ncu artifacts -- launch list of the bench command, ncu --set full of one config-5 GEMM band (fused tau_b epilogue)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/s5x_b.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5x_launches_config5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/s5x_ncu_launches.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 8 -c 1 -o gpurun_out/s5x_c5_gemm -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/s5x_ncu5.log 2>&1; echo ncu5=$?
ncu -i gpurun_out/s5x_c5_gemm.ncu-rep --page raw --csv > gpurun_out/s5x_c5_gemm_raw.csv 2>/dev/null
ls -la gpurun_out/s5x_*
