cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rank_rows -c 4 --csv --log-file gpurun_out/rank_launch.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rank_rows -c 2 --csv --log-file gpurun_out/rank_launch3.csv \
    python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_l3.log 2>&1; echo launches3=$?
