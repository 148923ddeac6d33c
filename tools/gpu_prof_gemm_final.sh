cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/run_path.py --config 2 --reps 2 > gpurun_out/plain_g.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_fp4 -s 1 -c 1 -o gpurun_out/prof_gemm_final -f \
    python tools/run_path.py --config 2 --reps 2 > gpurun_out/ncu_gf.log 2>&1; echo g=$?
