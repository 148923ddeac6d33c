cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=1 timeout 600 python tools/exp_plugin_c5.py 6 > gpurun_out/r2bn_c1.log 2>&1
timeout 300 python bench.py --config 1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 10 --e2e-tau-steps 3 > gpurun_out/r2bn_c1.json 2>&1
timeout 300 python bench.py --config 1 --steps 30 --warmup 5 --e2e-steps 3 --e2e-tau-steps 3 > gpurun_out/r2bn_c1_full.json 2>&1
