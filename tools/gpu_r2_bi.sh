# Final-state ncu --set full captures of the GEMM: config-5 row band 0, config 2, config 3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2bi_plain5.log 2>&1; echo plain5=$?
timeout 1200 ncu --set full --clock-control none -k regex:gemm_fp4 -c 1 -o gpurun_out/r2bi_c5_gemm -f \
    python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2bi_ncu5.log 2>&1; echo ncu5=$?
for c in 2 3; do
timeout 900 ncu --set full --clock-control none -k regex:gemm_fp4 -s 2 -c 1 -o gpurun_out/r2bi_c${c}_gemm -f \
    python tools/run_path.py --config $c --reps 3 > gpurun_out/r2bi_ncu$c.log 2>&1; echo ncu$c=$?
done
