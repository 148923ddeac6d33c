cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --graph off > gpurun_out/plain_c1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 14 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --graph off > gpurun_out/ncu_c1.log 2>&1; echo ncu=$?
