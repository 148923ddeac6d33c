# Merge-path iteration: merge parity tests, smoke, config-4 bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x -k "merge or config4 or smoke or engine" > gpurun_out/pytest_merge.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
