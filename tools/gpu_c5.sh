cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "config5 or gemm_splits or host_entry or config3" > gpurun_out/pt_c5.log 2>&1; echo pt=$?
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
