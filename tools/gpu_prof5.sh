cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 2 -c 1 -o gpurun_out/prof_gemm_fp4 \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_g.log 2>&1; echo full=$?
ncu --set full --clock-control none --import-source on -k regex:signpack -s 2 -c 1 -o gpurun_out/prof_signpack_fp4 \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_s.log 2>&1; echo full2=$?
