cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest_parity.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:signpack -s 1 -c 1 -o gpurun_out/prof_sp_v10 -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_sp.log 2>&1; echo full=$?
