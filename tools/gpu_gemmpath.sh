# GEMM-path iteration: GEMM-path parity tests and the config-2 bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not merge and not config4" > gpurun_out/pytest_gemm.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 100 --warmup 10 --e2e-steps 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:signpack -c 3 --csv --log-file gpurun_out/sp_time.csv python tools/run_path.py --config 2 --reps 3 > /dev/null 2>&1; echo ncu=$?
