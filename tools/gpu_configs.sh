# Bench lines for configs 1, 3, 5 (config 2 is the default bench; config 4 is the merge path)
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
