cd $GRAFT_REPO_ROOT
python tools/run_path.py --config 2 --reps 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"signpack" -s 1 -c 1 -o gpurun_out/prof_sp_v7 \
    python tools/run_path.py --config 2 --reps 2 > gpurun_out/ncu_sp.log 2>&1; echo ncu=$?
