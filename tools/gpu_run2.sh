cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_v2.log 2>&1; echo bench=$?
TB_GEMM_VARIANT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v1.log 2>&1; echo bench1=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
TB_GEMM_VARIANT=1 timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_c3_v1.log 2>&1; echo bench3v1=$?
