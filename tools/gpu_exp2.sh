cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x -k "merge or config4 or small_shapes or constant or corpus or boundary or host_entry" > gpurun_out/pytest_merge.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
