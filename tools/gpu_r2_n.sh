cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_n.log 2>&1; echo smoke=$?
timeout 300 python tools/run_path.py --config 4 --rows 64 --reps 1 > gpurun_out/r2_plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_pairs -c 1 -o gpurun_out/r2_k4 python tools/run_path.py --config 4 --rows 64 --reps 1 > gpurun_out/r2_ncu_k4.log 2>&1; echo ncu=$?
