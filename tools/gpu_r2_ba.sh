cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPLITS=0,24,32 timeout 300 python tools/exp_splits.py 1 > gpurun_out/r2ba_splits_c1.log 2>&1; echo s=$?
SPLITS=0,3 timeout 300 python tools/exp_splits.py 2 > gpurun_out/r2ba_splits_c2.log 2>&1; echo s=$?
timeout 300 python bench.py --config 1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2ba_c1.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "small_shapes or config1 or config2 or splits" > gpurun_out/r2ba_pt.log 2>&1; echo pt=$?
