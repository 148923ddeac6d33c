cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 --steps 30 --warmup 5 > gpurun_out/f6_bench_c1_rerun.json 2>&1; echo c1=$?
timeout 600 python bench.py --config 2 --steps 30 --warmup 5 > gpurun_out/f6_bench_c2_rerun.json 2>&1; echo c2=$?
