cd $GRAFT_REPO_ROOT
python tools/run_path.py --config 4 --rows 48 --reps 2 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 1 -c 1 -o gpurun_out/prof_merge_v3 \
    python tools/run_path.py --config 4 --rows 48 --reps 2 > gpurun_out/ncu_mg.log 2>&1; echo ncu_mg=$?
