# ncu evidence for the output write (K5 finalize) on configs 2 and 3, plus the config-4 launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/run_path.py --config 3 --reps 2 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:finalize_chunk -s 1 -c 1 -o gpurun_out/prof_fin_c3 -f \
    python tools/run_path.py --config 3 --reps 2 > gpurun_out/ncu_fin3.log 2>&1; echo fin3=$?
timeout 900 ncu --set full --clock-control none -k regex:finalize_chunk -s 1 -c 1 -o gpurun_out/prof_fin_c2 -f \
    python tools/run_path.py --config 2 --reps 2 > gpurun_out/ncu_fin2.log 2>&1; echo fin2=$?
timeout 900 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_c4.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_l4.log 2>&1; echo l4=$?
