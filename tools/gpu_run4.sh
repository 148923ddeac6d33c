cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
python tools/run_path.py --config 2 --reps 3 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:signpack -s 1 -c 1 -o gpurun_out/prof_signpack_v4 \
    python tools/run_path.py --config 2 --reps 3 > gpurun_out/ncu_sp.log 2>&1; echo ncu_sp=$?
python tools/run_path.py --config 4 --rows 48 --reps 2 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 1 -c 1 -o gpurun_out/prof_merge_v2 \
    python tools/run_path.py --config 4 --rows 48 --reps 2 > gpurun_out/ncu_mg.log 2>&1; echo ncu_mg=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_gemm_v2 \
    python tools/run_path.py --config 2 --reps 3 > gpurun_out/ncu_gm.log 2>&1; echo ncu_gm=$?
