cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x -k "host_entry or engine" > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2b.log 2>&1; echo bench=$?
