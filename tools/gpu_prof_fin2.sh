cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:finalize_chunk -s 1 -c 1 -o gpurun_out/prof_fin_c3b -f \
    python tools/run_path.py --config 3 --reps 2 > gpurun_out/ncu_fin3b.log 2>&1; echo fin3=$?
