cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/run_path.py --config 4 --rows 96 --reps 2 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 1 -c 1 -o gpurun_out/prof_merge_final -f \
    python tools/run_path.py --config 4 --rows 96 --reps 2 > gpurun_out/ncu_mg.log 2>&1; echo ncu_mg=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
