cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
