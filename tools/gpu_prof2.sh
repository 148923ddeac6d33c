cd $GRAFT_REPO_ROOT
python tools/run_path.py --config 2 --reps 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"signpack|rank_rows" -s 2 -c 2 -o gpurun_out/prof_sp_rk_v5 \
    python tools/run_path.py --config 2 --reps 2 > gpurun_out/ncu_sp.log 2>&1; echo ncu=$?
