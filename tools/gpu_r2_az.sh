cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPLITS=0,1,2,4,8,12,16,24,32,48,74 timeout 300 python tools/exp_splits.py 1 > gpurun_out/r2az_splits_c1.log 2>&1; echo s=$?
timeout 300 python bench.py --config 1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2az_c1_plain.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2az_launches_c1.csv \
   python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2az_ncu_c1.log 2>&1; echo n=$?
