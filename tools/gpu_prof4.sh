cd $GRAFT_REPO_ROOT
python tools/run_path.py --config 3 --reps 2 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"finalize" -s 1 -c 1 -o gpurun_out/prof_fin \
    python tools/run_path.py --config 3 --reps 2 > gpurun_out/ncu_fin.log 2>&1; echo ncu=$?
