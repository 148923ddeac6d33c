cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 2 -c 1 -o gpurun_out/prof_gemm_fp4_v6 -f \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_g.log 2>&1; echo full2=$?
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 1 -c 1 -o gpurun_out/prof_gemm_fp4_c3_v6 -f \
    python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_g3.log 2>&1; echo full3=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 14 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
