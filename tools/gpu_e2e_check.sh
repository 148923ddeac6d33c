cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "host_entry" > gpurun_out/pt_he.log 2>&1; echo pt=$?
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
