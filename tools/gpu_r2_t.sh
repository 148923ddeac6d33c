cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu_t.log 2>&1; echo pytest=$?
timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2_splits_c2_v3.log 2>&1
TB_GEMM_NO_FIXUP=1 timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2_splits_c2_v3_nofix.log 2>&1
for c in 2 1; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/r2_bench_c${c}_t.json 2>&1; done
