cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_engine.py -q -x --timeout 900 > gpurun_out/r2ao_pt_engine.log 2>&1; echo pt=$?
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2ao_c5.json 2>&1; echo c5=$?
