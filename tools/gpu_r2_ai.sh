cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/exp_plugin_c5.py 1000000 10 8 6 5 4 > gpurun_out/r2ai_plugin_c5.log 2>&1; echo exp=$?
for fe in 6 8; do
TB_RECORDS_FULL_EVERY=$fe timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --e2e-tau-steps 0 > gpurun_out/r2ai_c5_fe$fe.json 2> gpurun_out/r2ai_c5_fe$fe.err; echo c5=$?
done
