# Re-entry check: all GPU tests, smoke, default bench (config 2) and the merge-path bench (config 4).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
