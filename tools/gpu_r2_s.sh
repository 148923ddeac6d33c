cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2_splits_c2_v2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu_s.log 2>&1; echo pytest=$?
for c in 2 1; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/r2_bench_c${c}_s.json 2>&1; done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5_s.json 2>&1; echo c5=$?
