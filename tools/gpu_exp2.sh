cd $GRAFT_REPO_ROOT
TB_TRACE=1 timeout 300 python tools/exp_epi.py 2 3 > gpurun_out/exp_trace.log 2>&1; echo exp=$?
timeout 300 python tools/exp_epi.py 2 3 > gpurun_out/exp_epi.log 2>&1; echo exp=$?
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench=$?
