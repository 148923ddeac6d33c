# One GPU pass: all GPU tests, the default bench, its launch list, one full capture of the GEMM.
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 2 -c 1 -o gpurun_out/prof_gemm_fp4_v4 -f \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_g.log 2>&1; echo full=$?
