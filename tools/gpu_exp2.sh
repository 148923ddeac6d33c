cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --impl reference --config 3 --steps 2 --warmup 1 > gpurun_out/bench_ref3.log 2>&1; echo ref3=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
