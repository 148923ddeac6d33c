cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu_q.log 2>&1; echo pytest=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5_q.json 2>&1; echo c5=$?
timeout 600 python bench.py --config 1 --steps 30 --warmup 5 > gpurun_out/r2_bench_c1_q.json 2>&1; echo c1=$?
