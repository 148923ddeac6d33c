cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/run_path.py --config 1 --reps 20 > gpurun_out/r2_plain_c1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c1.csv python tools/run_path.py --config 1 --reps 20 > gpurun_out/r2_ncu_c1.log 2>&1; echo c1=$?
timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -k "config5_record" --timeout 900 > gpurun_out/r2_pytest_c5rec.log 2>&1; echo c5rec=$?
