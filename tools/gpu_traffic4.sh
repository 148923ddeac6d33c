cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:merge_pairs -s 1 -c 1 --csv \
    --log-file gpurun_out/traffic4.csv python tools/run_path.py --config 4 --reps 2 > gpurun_out/traffic4.log 2>&1; echo t4=$?
