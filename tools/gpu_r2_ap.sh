# K4 final-state ncu capture (config-4 rows 0..95).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/run_path.py --config 4 --rows 96 --reps 2 > gpurun_out/r2ap_plain4.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 1 -c 1 -o gpurun_out/r2ap_prof_merge -f \
    python tools/run_path.py --config 4 --rows 96 --reps 2 > gpurun_out/r2ap_ncu_mg.log 2>&1; echo ncu=$?
