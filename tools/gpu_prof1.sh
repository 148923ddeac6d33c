cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_v1.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu1.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_v1 \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu2.log 2>&1
echo full=$?
ncu --set full --clock-control none --import-source on -k regex:signpack -s 2 -c 1 -o gpurun_out/prof_signpack_v1 \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu3.log 2>&1
echo full2=$?
