# Hybrid record pipeline: engine GPU tests, then config-5 plugin e2e at several full/compact mixes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_engine.py -q -x --timeout 900 > gpurun_out/r2ad_pt_engine.log 2>&1; echo pt=$?
for fe in 1 3 10 1000000; do
  TB_RECORDS_FULL_EVERY=$fe timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 --e2e-tau-steps 0 > gpurun_out/r2ad_c5_fe$fe.json 2> gpurun_out/r2ad_c5_fe$fe.err; echo c5_fe$fe=$?
done
