cd $GRAFT_REPO_ROOT
timeout 900 python tools/exp_fp8.py 2 3 > gpurun_out/exp_fp8.log 2>&1; echo exp=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
python tools/run_path.py --config 2 --reps 3 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_v6.csv \
    python tools/run_path.py --config 2 --reps 3 > gpurun_out/ncu1.log 2>&1; echo launches=$?
