cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_v3.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu1.log 2>&1
echo launches=$?
