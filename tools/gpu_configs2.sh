# Refresh the bench lines of configs 1, 3, 5 and 2 (default) after kernel changes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
